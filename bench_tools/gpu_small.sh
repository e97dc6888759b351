cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TAG=${1:-sm}
for k in auto tiles dense; do for n in 3 6 9; do timeout 300 python bench.py --n $n --steps 5 --warmup 3 --no-cpu-baseline --kernel $k > gpurun_out/${TAG}_${k}_n$n.log 2>&1; done; done
for n in 3 6; do timeout 300 python bench.py --n $n --steps 5 --warmup 3 --no-cpu-baseline --no-symmetry > gpurun_out/${TAG}_nosym_n$n.log 2>&1; done
