TAG=r2r bash tools/gpu_tests.sh
TAG=r2s bash tools/gpu_round2.sh
