# Round profile evidence on one B200 (run after the plain commands exit 0 without ncu):
#   /usr/local/graft/bin/gpurun --timeout 2400 -- 'bash tools/profile_round.sh r02'
r=${1:-r02}
out=gpurun_out/prof_$r
mkdir -p $out
python bench.py --steps 50 --warmup 5 > $out/bench.json 2> $out/bench.err || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"quantize|router|topk|permute|to_umma|lut_umma|silu|combine|gather|row_sums" -c 40 --csv --log-file $out/launches_mx.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > /dev/null 2>&1
ncu --set full --import-source on --clock-control none -k regex:lut_umma_kernel -s 6 -c 2 -o $out/lut_umma_decode python bench.py --steps 2 --warmup 1 --no-cpu-baseline > /dev/null 2>&1
for c in ph qw ds mx1 qw64; do
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"quantize|router|topk|permute|to_umma|lut_umma|silu|combine|gather|row_sums|rot_|rq_|shared" -c 30 --csv --log-file $out/launches_$c.csv python bench.py --config $c --steps 1 --warmup 1 --no-cpu-baseline > /dev/null 2>&1
done
ncu --set full --import-source on --clock-control none -k regex:lut_umma_kernel -s 2 -c 2 -o $out/lut_umma_prefill_ph python bench.py --config ph --steps 1 --warmup 1 --no-cpu-baseline > /dev/null 2>&1
ls -la $out
