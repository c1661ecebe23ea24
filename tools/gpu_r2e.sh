mkdir -p gpurun_out
TAG=r2e PYTEST_ARGS="tests/test_gpu_states.py tests/test_gpu_multi.py tests/test_gpu_search.py tests/test_gpu_parity.py" bash tools/gpu_tests.sh
for lb in 256 2048 8192; do
  timeout 600 python bench.py --metric search --leaf-batch $lb --warmup 1 --no-cpu-baseline > gpurun_out/search_lb$lb.json 2> gpurun_out/search_lb$lb.err; echo "search lb=$lb rc=$?"; tail -c 600 gpurun_out/search_lb$lb.json
done
