#!/usr/bin/env bash
# compute-sanitizer over the layer kernel (tools/sanitize_run.py): memcheck,
# racecheck (shared-memory hazards), synccheck (barrier / mbarrier misuse).
# Logs go to gpurun_out/sanitize_<tool>.log; copy them under profiles/.
set -u
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for tool in memcheck racecheck synccheck; do
  timeout 1500 compute-sanitizer --tool "$tool" --kernel-name kns=layer_kernel \
      --print-limit 200 --error-exitcode 9 \
      python tools/sanitize_run.py > "gpurun_out/sanitize_${tool}.log" 2>&1
  echo "$tool rc=$?" | tee -a gpurun_out/sanitize_summary.txt
done
