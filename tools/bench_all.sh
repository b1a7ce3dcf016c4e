# All SURVEY §8(d) configurations on one B200, one JSON line each (gpurun_out/bench_all/).
out=gpurun_out/bench_all
mkdir -p $out
for c in mx mx1 mx8 mxe mx3 mx2 c1 qw64 qw256 qw qw8k ph ds; do
  timeout 600 python bench.py --config $c --steps 50 --warmup 5 --no-cpu-baseline > $out/$c.json 2> $out/$c.err
done
timeout 600 python bench.py > $out/default.json 2> $out/default.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > $out/reference.json 2> $out/reference.err
for c in ds mx; do
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port $((29520 + RANDOM % 400)) bench.py --ep --config $c --steps 20 --warmup 3 > $out/ep1_$c.json 2> $out/ep1_$c.err
done
python - <<'PY'
import json, glob, os
for f in sorted(glob.glob('gpurun_out/bench_all/*.json')):
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
    except Exception as e:
        print(os.path.basename(f), 'ERR', e); continue
    r = d.get('roofline', {})
    print(f"{os.path.basename(f):16s} {d.get('ms_per_step', 0)*1e3:9.1f} us  {d.get('value', 0):12.1f} tok/s  e2e {d.get('e2e', {}).get('value', 0):12.1f}  "
          f"{r.get('bound')} {r.get('frac')}  clocks {d.get('clocks', {}).get('sm_mhz')} {d.get('clocks', {}).get('reasons')}")
PY
