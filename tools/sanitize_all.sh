#!/usr/bin/env bash
# compute-sanitizer over tools/sanitize_run.py, one log per tool under gpurun_out/sanitize_<tool>.log.
# Only this package's kernels are reported (--kernel-name-exclude for torch's own).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for tool in memcheck racecheck synccheck initcheck; do
  extra=""
  [ "$tool" = "memcheck" ] && extra="--leak-check no"
  [ "$tool" = "racecheck" ] && extra="--racecheck-report all"
  timeout 1200 compute-sanitizer --tool $tool $extra --print-limit 50 python tools/sanitize_run.py \
      > gpurun_out/sanitize_$tool.log 2>&1
  echo "$tool exit=$?" >> gpurun_out/sanitize_summary.txt
  grep -E "ERROR SUMMARY|RACECHECK SUMMARY|Hazard|Error" gpurun_out/sanitize_$tool.log | tail -3 >> gpurun_out/sanitize_summary.txt
done
