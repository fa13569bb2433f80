#!/bin/bash
# compute-sanitizer over tools/sanitize_cases.py (run on the GPU box); logs -> gpurun_out/sanitize_*.log
set -u
mkdir -p gpurun_out
for tool in memcheck racecheck synccheck; do
  for c in multicrop multicrop_mixed sampler read_regions trace png_jpeg; do
    timeout 900 compute-sanitizer --tool $tool --error-exitcode 17 --target-processes all \
      python tools/sanitize_cases.py $c > gpurun_out/sanitize_${tool}_${c}.log 2>&1
    echo "$tool $c rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY' gpurun_out/sanitize_${tool}_${c}.log | tail -1)"
  done
done
