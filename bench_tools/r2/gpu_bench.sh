# bench lines for several n on one B200 (after the tests); logs under gpurun_out/<tag>_*
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TAG=${1:-r2}
shift
for n in ${@:-3 6 9 12}; do
  timeout 600 python bench.py --n $n --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/${TAG}_bench_n$n.log 2>&1
done
