# row-grouping window (greedy tiles) 256 / 512 / 1024 rows at n = 12 and n = 11
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TAG=${1:-win}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${TAG}_build.log 2>&1
python bench_tools/build_variants.py w512=-DMP_GRP_WIN=512 w1024=-DMP_GRP_WIN=1024 >> gpurun_out/${TAG}_build.log 2>&1
for n in 12 11; do
  timeout 300 python bench.py --n $n --no-cpu-baseline > gpurun_out/${TAG}_n${n}.log 2>&1
  for v in w512 w1024; do
    MP_LIB_PATH=bench_tools/variants/$v.so timeout 300 python bench.py --n $n --no-cpu-baseline > gpurun_out/${TAG}_n${n}_$v.log 2>&1
  done
done
