mkdir -p gpurun_out
for i in 1 2; do python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-parity-sample 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('cfg3', d['value'], d['ms_per_step'], d['config']['arena_bytes'])"; done
timeout 900 python bench.py --config 4 --sizes 16384 --steps 1 --warmup 1 --no-cpu-baseline --p1-parents 4 > gpurun_out/cfg4_r2l.json 2> gpurun_out/cfg4_r2l.err; echo "sweep rc=$?"; python -c "import json; d=json.load(open('gpurun_out/cfg4_r2l.json')); print(d['config']['arena_bytes'], d['config']['slots'], d['sweep'])"
