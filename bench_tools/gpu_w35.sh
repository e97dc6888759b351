cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for n in 3 6 9 12; do timeout 300 python bench.py --n $n --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/w35_bench_n$n.log 2>&1; done
