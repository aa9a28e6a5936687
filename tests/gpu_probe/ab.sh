#!/bin/bash
# Interleaved A/B of library variants (make variant VNAME=<name> VFLAGS=...) on one config:
#   bash tests/gpu_probe/ab.sh <config> <rounds> base <variant> [<variant> ...]
# "base" is the product library; every other name loads _lib/libflashbias_b200_<name>.so.
CFG=$1; ROUNDS=$2; shift 2
for r in $(seq 1 "$ROUNDS"); do
  for v in "$@"; do
    if [ "$v" = base ]; then
      timeout 300 python tests/gpu_probe/fwd_bwd_time.py "$CFG"
    else
      FLASHBIAS_B200_VARIANT=$v timeout 300 python tests/gpu_probe/fwd_bwd_time.py "$CFG"
    fi
  done
done
