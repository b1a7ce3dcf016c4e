mkdir -p gpurun_out/ep1
timeout 900 python -m pytest tests/test_gpu_ep.py -q -x -p no:cacheprovider --durations=10 > gpurun_out/ep1/pytest.log 2>&1; echo "rc $?" >> gpurun_out/ep1/pytest.log
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29511 bench.py --ep --steps 50 --warmup 5 > gpurun_out/ep1/bench_mx_ep1.json 2> gpurun_out/ep1/bench_mx_ep1.err
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29512 bench.py --ep --config ds --steps 20 --warmup 3 > gpurun_out/ep1/bench_ds_ep1.json 2> gpurun_out/ep1/bench_ds_ep1.err
tail -3 gpurun_out/ep1/pytest.log; cat gpurun_out/ep1/*.json; tail -5 gpurun_out/ep1/*.err
