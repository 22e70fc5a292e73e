#!/usr/bin/env bash
# Round-end style checks on one GPU: smoke(), torchrun (1 rank) bench, and
# the profiles of configs 3 / 4 / 5 (launch list + one full capture each).
set -u
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -2
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29512 \
  bench.py --gpus 1 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/torchrun1.log 2>&1
echo "torchrun rc=$?"; tail -c 400 gpurun_out/torchrun1.log
bash tools/profile_round.sh 3 r01 maxvol_large_kernel tsqr_reduce_kernel
bash tools/profile_round.sh 4 r01 lsr_residual_kernel cholesky_kernel
