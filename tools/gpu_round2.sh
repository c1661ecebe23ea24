#!/bin/bash
# Round-2 measurement session: headline bench, launch list, one ncu --set full
# capture of the main rollout launch, config-4 sweep, search metric, reference arms.
mkdir -p gpurun_out
T=${TAG:-r2m}
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_$T.json 2> gpurun_out/bench_$T.err; echo "bench rc=$?"
SMALL="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-parity-sample"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${T}_launches.csv $SMALL > gpurun_out/${T}_ncu_launch.log 2>&1; echo "launch list rc=$?"
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:pe_rollout_kernel -s 8 -c 3 -o gpurun_out/${T}_full -f $SMALL > gpurun_out/${T}_ncu_full.log 2>&1; echo "ncu full rc=$?"
ncu -i gpurun_out/${T}_full.ncu-rep --page raw --csv > gpurun_out/${T}_full_raw.csv 2>/dev/null; echo "export rc=$?"
timeout 600 python bench.py --metric search --leaf-batch 256 --warmup 1 > gpurun_out/search_$T.json 2> gpurun_out/search_$T.err; echo "search rc=$?"
timeout 900 python bench.py --impl reference --steps 10 --warmup 3 > gpurun_out/ref_$T.json 2> gpurun_out/ref_$T.err; echo "ref rc=$?"
timeout 2400 python bench.py --config 4 --sizes 1024,4096,16384,65536,262144,1048576 --steps 1 --warmup 1 --cpu-cap-s 120 > gpurun_out/cfg4_$T.json 2> gpurun_out/cfg4_$T.err; echo "cfg4 rc=$?"
