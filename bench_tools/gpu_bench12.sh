# bench only (n = 11, 12), no tests: quick kernel timing
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TAG=${1:-b}
for n in 11 12; do timeout 300 python bench.py --n $n --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/${TAG}_bench_n$n.log 2>&1; done
