# small-N path: warps per CTA (MP_SMALL_WARPS) at n = 3 and n = 6; small-path tests
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TAG=${1:-small}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${TAG}_build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_small.py -x -q --timeout 300 > gpurun_out/${TAG}_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/${TAG}_pytest.log
for n in 3 6; do
  timeout 300 python bench.py --n $n --no-cpu-baseline > gpurun_out/${TAG}_n$n.log 2>&1
  for w in 1 2 4 8 16; do MP_SMALL_WARPS=$w timeout 300 python bench.py --n $n --no-cpu-baseline > gpurun_out/${TAG}_n${n}_w$w.log 2>&1; done
done
MP_SMALL_WARPS=1 timeout 600 python -m pytest tests/test_gpu_small.py -x -q --timeout 300 > gpurun_out/${TAG}_pytest_w1.log 2>&1; echo "rc=$?" >> gpurun_out/${TAG}_pytest_w1.log
