# k_spmm variants at n = 12 through MP_LIB_PATH (the product .so is never overwritten)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TAG=${1:-var}
shift
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${TAG}_build.log 2>&1
timeout 300 python bench.py --n 12 --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/${TAG}_base.log 2>&1
for v in "$@"; do
  MP_LIB_PATH=bench_tools/variants/$v.so timeout 300 python bench.py --n 12 --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/${TAG}_$v.log 2>&1
done
for w in -512 512; do
  timeout 300 python bench.py --n 12 --steps 2 --warmup 1 --no-cpu-baseline --spmm-width $w > gpurun_out/${TAG}_w$w.log 2>&1
done
timeout 600 python bench_tools/oracle_runs.py gpurun_out/${TAG}_oracle_runs.json 9 10 > gpurun_out/${TAG}_oracle_runs.log 2>&1
for n in 3 6 9; do timeout 300 python bench.py --n $n --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/${TAG}_bench_n$n.log 2>&1; done
timeout 600 python -m pytest tests/test_gpu_small.py -x -q > gpurun_out/${TAG}_pytest_small.log 2>&1; echo "rc=$?" >> gpurun_out/${TAG}_pytest_small.log
