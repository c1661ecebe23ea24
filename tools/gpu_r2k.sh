mkdir -p gpurun_out
TAG=r2k PYTEST_ARGS="tests/test_gpu_bounds.py tests/test_gpu_parity.py tests/test_gpu_infer_rest.py tests/test_gpu_states.py tests/test_graph_loader.py" bash tools/gpu_tests.sh
timeout 900 python bench.py --config 4 --sizes 16384 --steps 1 --warmup 1 --no-cpu-baseline --p1-parents 4 > gpurun_out/cfg4_r2k.json 2> gpurun_out/cfg4_r2k.err; echo "sweep rc=$?"; python -c "import json; d=json.load(open('gpurun_out/cfg4_r2k.json')); print(d['config'], d['sweep'])"
