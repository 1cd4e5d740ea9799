#!/bin/bash
# compute-sanitizer over every kernel family; logs to gpurun_out/sanitize_*.log
cd "$(dirname "$0")/.."
CS=/usr/local/cuda/bin/compute-sanitizer
mkdir -p gpurun_out
for tool in memcheck racecheck synccheck; do
  for part in fused split verify; do
    timeout 1200 $CS --tool $tool --print-limit 20 python tools/sanitize_driver.py $part > gpurun_out/sanitize_${tool}_${part}.log 2>&1
    echo "$tool $part rc $?" >> gpurun_out/sanitize_summary.txt
    tail -3 gpurun_out/sanitize_${tool}_${part}.log >> gpurun_out/sanitize_summary.txt
  done
done
