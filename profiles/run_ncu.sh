#!/bin/bash
# Profiling recipe used for profiles/ (run under gpurun on one B200).
# 1) launch list with device times of one C3 bench step (cold-cache, serialised)
# 2) one full-set capture of each FlashBias kernel (fwd K1, fused 128x128-tile bwd K2)
set -e
mkdir -p gpurun_out
TAG=${1:-r01}
ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches_${TAG}.csv \
    python bench.py --config C3 --steps 1 --warmup 1 --skip-dense --skip-e2e --skip-cpu > gpurun_out/launches_${TAG}.log 2>&1
for K in fb_fwd_kernel fb_bwd_t128_kernel; do
  ncu --set full --clock-control none --import-source on -k regex:${K} -s 1 -c 1 \
      -o gpurun_out/prof_${TAG}_${K} -f \
      python bench.py --config C3 --steps 1 --warmup 1 --skip-dense --skip-e2e --skip-cpu > /dev/null 2>&1 || true
done
