mkdir -p gpurun_out
TAG=r2g PYTEST_ARGS="tests/test_gpu_cfg4_golden.py" bash tools/gpu_tests.sh
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_r2g.json 2> gpurun_out/bench_r2g.err; echo "bench rc=$?"
cat gpurun_out/bench_r2g.json
