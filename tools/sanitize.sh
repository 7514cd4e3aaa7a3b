#!/bin/bash
# compute-sanitizer over tools/sanitize_cases.py (every hot kernel on small ragged shapes);
# logs to gpurun_out/sanitize_<tool>.log.  Usage (GPU box): bash tools/sanitize.sh
mkdir -p gpurun_out
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck racecheck synccheck initcheck; do
  timeout 900 $CS --tool $tool --target-processes all --print-limit 50 \
    python tools/sanitize_cases.py > gpurun_out/sanitize_$tool.log 2>&1
  echo "$tool rc=$?" >> gpurun_out/sanitize_$tool.log
  tail -3 gpurun_out/sanitize_$tool.log
done
