#!/bin/bash
# Profiling recipe used for profiles/ (run under gpurun on one B200).
#   bash profiles/run_ncu.sh <tag> <config> [extra bench.py args]
# 1) launch list with device times of the bench steps of <config> (cold-cache, serialised)
# 2) one --set full capture of the step's forward kernel and of its backward kernel
set -e
mkdir -p gpurun_out
TAG=${1:-r02}
CFG=${2:-C3}
shift 2 || true
ARGS="--config $CFG --steps 1 --warmup 1 --skip-dense --skip-e2e --skip-cpu --skip-sdpa --ref-svd-heads 0 --no-graph $*"
# only the timed bench steps are profiled (BENCH_PROFILE_RANGE=1 brackets them with cudaProfilerStart/Stop), so the
# setup (input generation, the device SVD of C4/C5: cuSOLVER kernels ncu cannot replay) stays outside
export BENCH_PROFILE_RANGE=1
ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches_${TAG}_${CFG}.csv python bench.py $ARGS > gpurun_out/launches_${TAG}_${CFG}.log 2>&1
KS='fb_fwd_kernel "fb_bwd_(t128|fused|fused64|dkv)_kernel"'
[ "$CFG" = C1 ] && KS=fwd_simt_tiled_kernel  # the fp32 SIMT forward is the whole C1 step
eval "set -- $KS"
for K in "$@"; do
  NAME=$( [ "$K" = "fb_bwd_(t128|fused|fused64|dkv)_kernel" ] && echo bwd || echo fwd )
  ncu --profile-from-start off --set full --clock-control none --import-source on -k "regex:${K}" -s 1 -c 1 \
      -o gpurun_out/prof_${TAG}_${CFG}_${NAME} -f python bench.py $ARGS > /dev/null 2>&1 || true
  # gpurun copies back <= 64 MiB: keep the raw-page CSV (what summarize.py reads), drop the report unless asked
  if [ -f gpurun_out/prof_${TAG}_${CFG}_${NAME}.ncu-rep ]; then
    ncu -i gpurun_out/prof_${TAG}_${CFG}_${NAME}.ncu-rep --page raw --csv > gpurun_out/prof_${TAG}_${CFG}_${NAME}.raw.csv
    [ -n "${KEEP_REP:-}" ] || rm -f gpurun_out/prof_${TAG}_${CFG}_${NAME}.ncu-rep
  fi
done
