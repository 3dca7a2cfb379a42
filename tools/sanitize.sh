#!/usr/bin/env bash
# GPU box: compute-sanitizer memcheck / racecheck / synccheck over tools/sanitize_kernels.py with
# each attention backend; logs into gpurun_out/sanitize_<tool>_<backend>.log (summarised into
# profiles/r02_sanitizer.md).
set -u
mkdir -p gpurun_out
for tool in memcheck synccheck racecheck; do
  for be in tc tp fa mma; do
    TA_ATTENTION_BACKEND=$be timeout 900 compute-sanitizer --tool $tool --target-processes all \
      python tools/sanitize_kernels.py > gpurun_out/sanitize_${tool}_${be}.log 2>&1
    echo "$tool $be rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|all launches done' gpurun_out/sanitize_${tool}_${be}.log | tr '\n' ' ')"
  done
done
