# Same-box A/B of two builds of libcq_b200.so (whole steps): build the baseline and the candidate
# into abtest/base.so and abtest/new.so (e.g. `make BUILD=build_x OUT=../../abtest/new.so DEFS=...`
# in paper_2604_10496_b200/csrc), then on the GPU:  bash tools/ab.sh "cfg1 cfg2" [steps]
# Three alternations of base / new per config (box-to-box spread is larger than most changes).
cfgs=${1:-"ph ds"}; steps=${2:-30}
for rep in 1 2 3; do for v in base new; do for c in $cfgs; do
  CQ_B200_LIB=abtest/$v.so timeout 600 python bench.py --config $c --steps $steps --warmup 5 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', '$c', round(d['ms_per_step']*1e3,1), d['clocks']['reasons'])"
done; done; done
