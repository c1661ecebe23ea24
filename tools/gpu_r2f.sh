mkdir -p gpurun_out
TAG=r2f PYTEST_ARGS="tests/test_gpu_launch_shape.py -k config4" bash tools/gpu_tests.sh
timeout 900 python bench.py --config 4 --sizes 1024,4096 --steps 1 --warmup 1 --cpu-cap-s 20 --p1-parents 16 > gpurun_out/cfg4_r2f.json 2> gpurun_out/cfg4_r2f.err; echo "sweep rc=$?"
tail -5 gpurun_out/cfg4_r2f.err; cat gpurun_out/cfg4_r2f.json
