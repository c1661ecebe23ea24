#!/bin/bash
# One GPU session: bench line, launch list, one ncu --set full capture.
set -x
mkdir -p gpurun_out
TAG=${TAG:-r1}
python bench.py --steps ${STEPS:-10} --warmup 3 > gpurun_out/bench_${TAG}.json 2> gpurun_out/bench_${TAG}.err; echo "bench rc=$?"
SMALL="python bench.py --steps 2 --warmup 1 --batch ${NCU_BATCH:-16384} --no-cpu-baseline"
$SMALL > gpurun_out/plain_${TAG}.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${TAG}.csv $SMALL > gpurun_out/ncu_launch_${TAG}.log 2>&1; echo "launch rc=$?"
if [ "${FULL:-1}" = "1" ]; then
ncu --set full --clock-control none --import-source on -k regex:pe_rollout -s 2 -c 1 -o gpurun_out/prof_${TAG} -f $SMALL > gpurun_out/ncu_full_${TAG}.log 2>&1; echo "full rc=$?"
fi
