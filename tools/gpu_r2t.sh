TAG=r2t PYTEST_ARGS="tests/test_gpu_states.py tests/test_gpu_search.py tests/test_gpu_parity.py -k trie_sched_or_states_or_search_or_prefix" bash tools/gpu_tests.sh
TAG=r2t PYTEST_ARGS="tests/test_gpu_states.py tests/test_gpu_search.py tests/test_gpu_cfg4_golden.py" bash tools/gpu_tests.sh
TAG=r2t2 PYTEST_ARGS="tests/test_gpu_parity.py -k trie" bash tools/gpu_tests.sh
timeout 900 python bench.py --config 4 --sizes 4096 --steps 1 --warmup 1 --no-cpu-baseline --p1-parents 64 2>&1 | grep parents
python bench.py --metric search --leaf-batch 256 --warmup 1 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('search', d['value'], d['prefix_cache'])"
