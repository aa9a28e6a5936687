set -u
mkdir -p gpurun_out
b() { n=$1; shift; timeout 900 python bench.py "$@" > gpurun_out/bench_r02c_$n.json 2> gpurun_out/bench_r02c_$n.err; echo "$n rc=$?"; }
b C3L --config C3 --steps 5 --warmup 3 --learnable --skip-e2e --skip-sdpa --skip-cpu
b C5r8L --config C5 --steps 5 --warmup 3 --rank 8 --learnable --skip-e2e --skip-sdpa --skip-cpu --ref-svd-heads 0
b C5r16L --config C5 --steps 5 --warmup 3 --rank 16 --learnable --skip-e2e --skip-sdpa --skip-cpu --ref-svd-heads 0
for C in C3 C4 C5; do timeout 700 bash profiles/run_ncu.sh r02c $C; done
timeout 700 bash profiles/run_ncu.sh r02cL C5 --learnable --rank 8
du -sh gpurun_out
