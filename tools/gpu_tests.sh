# GPU test suite on the box: TAG names the log
mkdir -p gpurun_out
TAG=${TAG:-x}
timeout ${TMO:-1500} python -m pytest tests -m gpu -q -p no:cacheprovider ${PYTEST_ARGS} > gpurun_out/gpu_tests_${TAG}.log 2>&1; echo "tests rc=$?"
tail -15 gpurun_out/gpu_tests_${TAG}.log
