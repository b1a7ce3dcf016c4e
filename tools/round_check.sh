# Round-end checks on one B200: the GPU test suite, smoke(), the default bench and the reference arm.
# /usr/local/graft/bin/gpurun --timeout 2400 -- 'bash tools/round_check.sh'
mkdir -p gpurun_out/final
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/final/pytest.log 2>&1; echo "pytest rc $?" >> gpurun_out/final/pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/final/smoke.log 2>&1
timeout 600 python bench.py > gpurun_out/final/bench.json 2> gpurun_out/final/bench.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/final/ref.json 2> gpurun_out/final/ref.err
