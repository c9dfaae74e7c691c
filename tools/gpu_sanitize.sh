#!/bin/bash
# compute-sanitizer over small invocations of every kernel family (summaries -> gpurun_out/sanitize_*.txt)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck racecheck synccheck initcheck; do
  for what in persist layered encoder refine; do
    timeout 900 $CS --tool $tool --print-limit 20 --error-exitcode 9 python tools/sanitize_run.py $what > gpurun_out/sanitize_${tool}_${what}.txt 2>&1
    echo "$tool $what rc=$?  $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|sanitize run ok' gpurun_out/sanitize_${tool}_${what}.txt | tr '\n' ' ')"
  done
done
