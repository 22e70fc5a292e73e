#!/usr/bin/env bash
# Profile capture for one round (run under gpurun, one GPU):
#   1. the bench command must exit 0 without ncu first;
#   2. launch list (gpu__time_duration per launch, our kernels only);
#   3. one `ncu --set full` capture per dominant kernel.
# Outputs land in gpurun_out/; tools/summarize_profiles.py turns them into
# the tracked summaries under profiles/.
set -u
CFG=${1:-2}
TAG=${2:-r01}
source tools/my_kernels.sh
BENCH="python bench.py --config $CFG --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 0"
$BENCH > gpurun_out/${TAG}_c${CFG}_bench.log 2>&1 || { echo "bench failed"; exit 1; }
ncu --metrics gpu__time_duration.sum --clock-control none --kernel-name-base function -k "$MYK" -c 400 --csv \
  --log-file gpurun_out/${TAG}_c${CFG}_launches.csv $BENCH > gpurun_out/${TAG}_c${CFG}_ncu_launch.log 2>&1
echo "launch list rc=$?"
shift 2 || true
for k in "$@"; do
  timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base function -k "regex:^$k" -c 1 \
    -o gpurun_out/${TAG}_c${CFG}_full_$k $BENCH > gpurun_out/${TAG}_c${CFG}_ncu_$k.log 2>&1
  echo "$k rc=$?"
done
