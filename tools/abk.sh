# Kernel-level A/B of two library builds (abtest/base.so, abtest/new.so; see tools/ab.sh): ncu launch
# times (cold caches, serialized) of the kernels matching a regex:  bash tools/abk.sh <regex> "cfg1 cfg2"
k=$1; cfgs=${2:-"ph ds"}
for v in base new; do for c in $cfgs; do
  CQ_B200_LIB=abtest/$v.so ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"$k" -c 4 --csv --log-file /tmp/abk_${v}_${c}.csv python bench.py --config $c --steps 1 --warmup 1 --no-cpu-baseline > /dev/null 2>&1
  echo "$v $c $(grep -h gpu__time /tmp/abk_${v}_${c}.csv | awk -F, '{print $NF}' | tr '\n' ' ')"
done; done
