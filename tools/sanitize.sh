#!/usr/bin/env bash
# compute-sanitizer over tools/sanitize_cases.py (every kernel family at small
# sizes): memcheck (+ leak check), racecheck (shared-memory hazards),
# synccheck (barrier misuse), initcheck (reads of uninitialised device
# memory). Writes gpurun_out/sanitize_<tool>.log; prints one summary line per
# tool. Run on the GPU box: gpurun -- bash tools/sanitize.sh [cases...]
set -u
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck racecheck synccheck initcheck; do
  extra=""
  [ $tool = memcheck ] && extra="--leak-check full"
  [ $tool = racecheck ] && extra="--racecheck-report hazard"
  timeout 1500 $CS --tool $tool $extra --target-processes all --error-exitcode 99 \
    python tools/sanitize_cases.py "$@" > gpurun_out/sanitize_$tool.log 2>&1
  rc=$?
  echo "$tool rc=$rc: $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|LEAK SUMMARY' gpurun_out/sanitize_$tool.log | tr '\n' ' ') cases: $(grep -c 'ok$' gpurun_out/sanitize_$tool.log)"
done
