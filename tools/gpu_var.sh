TAG=r2v PYTEST_ARGS="tests/test_gpu_parity.py tests/test_gpu_infer_rest.py tests/test_gpu_states.py tests/test_gpu_search.py tests/test_gpu_launch_shape.py tests/test_gpu_edges.py" bash tools/gpu_tests.sh
for B in 1 32 1024 4096; do for co in 0 1; do PE_COOP=$co WARM=3 B=$B CFG=3 python tools/variant_bench.py variants/coop.so 2>&1 | tail -1 | sed "s/^/cfg3 coop=$co B=$B /"; done; done
for co in 0 1; do PE_COOP=$co WARM=1 B=4096 CFG=4 python tools/variant_bench.py variants/coop.so 2>&1 | tail -1 | sed "s/^/cfg4 coop=$co /"; done
for co in 0 1; do PE_COOP=$co python bench.py --metric search --leaf-batch 256 --warmup 1 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('search coop=$co', d['value'], d['episodes_per_s_full_budget'])"; done
