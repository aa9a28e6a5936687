#!/bin/bash
# Round sweep (one B200, under gpurun): the bench line of every BASELINE config plus the
# learnable-factor and C5 rank-sweep variants, then (optionally) the ncu recipe per config.
#   bash profiles/run_sweep.sh <tag> [ncu]
# Outputs: gpurun_out/bench_<tag>_<name>.json (one JSON line each), gpurun_out/launches_* and
# gpurun_out/prof_*.ncu-rep when "ncu" is given (summarise with profiles/summarize.py <tag> <cfg>).
set -u
mkdir -p gpurun_out
TAG=${1:-r02}
NCU=${2:-}
run() {  # name, bench args...
  local name=$1; shift
  timeout 900 python bench.py "$@" > gpurun_out/bench_${TAG}_${name}.json 2> gpurun_out/bench_${TAG}_${name}.err
  echo "$name rc=$? $(head -c 300 gpurun_out/bench_${TAG}_${name}.json)"
}
run C3 --config C3
run C1 --config C1 --steps 20 --warmup 5
run C2 --config C2 --steps 20 --warmup 5
run C2s --config C2 --steps 20 --warmup 5 --static-factors
run C4 --config C4 --steps 20 --warmup 5
run C4r16 --config C4 --steps 20 --warmup 5 --rank 16
for R in 8 16 32 64; do run C5r$R --config C5 --steps 5 --warmup 3 --rank $R --skip-e2e; done
run C5 --config C5 --steps 10 --warmup 3
run C5L --config C5 --steps 5 --warmup 3 --learnable --skip-e2e --skip-sdpa
run C3L --config C3 --steps 5 --warmup 3 --learnable --skip-e2e --skip-sdpa
run MIX --config MIX --steps 20 --warmup 5
run ref --impl reference --steps 2 --warmup 0
if [ "$NCU" = ncu ]; then
  for CFG in C3 C2 C4 C5 C1; do timeout 900 bash profiles/run_ncu.sh "$TAG" "$CFG"; done
fi
