#!/bin/bash
# compute-sanitizer passes over tools/sanitize_workload.py; logs in gpurun_out/sanitize/
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out/sanitize
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck synccheck racecheck initcheck; do
  for part in ref grid rgg query; do
    timeout 900 $CS --tool $tool --print-limit 50 --error-exitcode 9 \
      python tools/sanitize_workload.py $part > gpurun_out/sanitize/${tool}_${part}.log 2>&1
    echo "$tool $part rc=$?" | tee -a gpurun_out/sanitize/summary.txt
  done
done
