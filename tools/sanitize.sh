#!/bin/bash
# compute-sanitizer over every engine kernel (tools/sanitize_workload.py);
# logs under gpurun_out/sanitize_*.log
mkdir -p gpurun_out
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck synccheck racecheck; do
  timeout 1500 $CS --tool $tool --print-limit 20 --error-exitcode 9 python tools/sanitize_workload.py > gpurun_out/sanitize_$tool.log 2>&1
  echo "$tool rc=$?"; tail -3 gpurun_out/sanitize_$tool.log
done
# the launch shape beyond the resident slots (SM-wide blocks, warp-chunked waves)
timeout 1500 $CS --tool synccheck --print-limit 20 --error-exitcode 9 python tools/sanitize_workload.py 1 > gpurun_out/sanitize_synccheck_big.log 2>&1
echo "synccheck big rc=$?"; tail -3 gpurun_out/sanitize_synccheck_big.log
timeout 1500 $CS --tool memcheck --print-limit 20 --error-exitcode 9 python tools/sanitize_workload.py 1 > gpurun_out/sanitize_memcheck_big.log 2>&1
echo "memcheck big rc=$?"; tail -3 gpurun_out/sanitize_memcheck_big.log
