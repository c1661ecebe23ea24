#!/bin/bash
# Round-2 final headline session at the 1,048,576-rollout step: bench, launch
# list, one ncu --set full capture of the main rollout launch (traffic).
mkdir -p gpurun_out
T=${TAG:-r2f}
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_$T.json 2> gpurun_out/bench_$T.err; echo "bench rc=$?"
SMALL="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-parity-sample --also-batch 0"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${T}_launches.csv $SMALL > gpurun_out/${T}_ncu_launch.log 2>&1; echo "launch list rc=$?"
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:pe_rollout_kernel -s 8 -c 3 -o gpurun_out/${T}_full -f $SMALL > gpurun_out/${T}_ncu_full.log 2>&1; echo "ncu full rc=$?"
ncu -i gpurun_out/${T}_full.ncu-rep --page raw --csv > gpurun_out/${T}_full_raw.csv 2>/dev/null; echo "export rc=$?"
