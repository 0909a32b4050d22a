#!/bin/bash
# Two-rank smoke of the multi-GPU round (needs 2 GPUs): NCCL communicator bootstrap, the
# partial -> allreduce -> finalize aggregation, stats gathered over ranks, oracle parity.
set -e
cd "$(dirname "$0")/.."
NCCL_DEBUG=${NCCL_DEBUG:-INFO} NCCL_DEBUG_SUBSYS=INIT,NVLS python -m torch.distributed.run --nnodes=1 \
  --nproc-per-node 2 --master-addr 127.0.0.1 --master-port ${PORT:-29511} scripts/dist_round_check.py
python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
  --master-port $(( ${PORT:-29511} + 1 )) bench.py --gpus 2 --steps 3 --warmup 3 --no-e2e
