#!/usr/bin/env bash
# Scaling recipe: C3 (or $CONFIG) on 1, 2, 4, 8 GPUs of one node, one rank per
# GPU over NCCL, B*H head-sharded with no collective in the timed region.  Each JSON line
# carries "collective": {"backend": "nccl", "nranks": N, "nccl_version": ...}.
#   bash profiles/run_scale.sh [C3] > profiles/scale_<round>.jsonl
set -euo pipefail
CONFIG=${1:-C3}
cd "$(dirname "$0")/.."
for N in 1 2 4 8; do
  if [ "$N" -eq 1 ]; then
    python bench.py --config "$CONFIG" --gpus 1 --steps 20 --warmup 5
  else
    python -m torch.distributed.run --nnodes=1 --nproc-per-node "$N" --master-addr 127.0.0.1 \
      --master-port $((29500 + N)) bench.py --config "$CONFIG" --gpus "$N" --steps 20 --warmup 5
  fi
done
