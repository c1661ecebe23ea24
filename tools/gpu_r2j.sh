mkdir -p gpurun_out
python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-parity-sample 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('cfg3', d['value'], d['ms_per_step'], d['config']['arena_bytes'])"
timeout 900 python bench.py --config 4 --sizes 16384 --steps 1 --warmup 1 --no-cpu-baseline --p1-parents 4 > gpurun_out/cfg4_r2j.json 2> gpurun_out/cfg4_r2j.err; echo "sweep rc=$?"; tail -3 gpurun_out/cfg4_r2j.err | cut -c1-300
TAG=r2j PYTEST_ARGS="tests/test_gpu_parity.py tests/test_gpu_launch_shape.py -k not_config4 tests/test_gpu_infer_rest.py tests/test_gpu_states.py" bash tools/gpu_tests.sh
