TAG=r2u bash tools/gpu_tests.sh
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_r2u.json 2> gpurun_out/bench_r2u.err; echo "bench rc=$?"; cat gpurun_out/bench_r2u.json | cut -c1-400
