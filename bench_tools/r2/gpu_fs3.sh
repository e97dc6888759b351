cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TAG=${1:-fs3}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${TAG}_build.log 2>&1
timeout 1500 python -m pytest tests/test_gpu_fullsize.py tests/test_gpu_small.py tests/test_gpu_multiprocess.py -x -q -k "not streamed" > gpurun_out/${TAG}_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/${TAG}_pytest.log
for n in 12 11 10; do
  timeout 600 python bench.py --n $n --no-cpu-baseline > gpurun_out/${TAG}_bench_n$n.log 2>&1
  MP_FOLD_STATS=0 timeout 600 python bench.py --n $n --no-cpu-baseline > gpurun_out/${TAG}_bench_n${n}_sep.log 2>&1
done
for n in 3 6; do MP_SMALL_PROFILE=1 timeout 300 python bench.py --n $n --no-cpu-baseline > gpurun_out/${TAG}_bench_n$n.log 2>&1; done
