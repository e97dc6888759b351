# small-N path: tests, bench at n = 3 and n = 6 (optionally MP_SMALL_WARPS=w)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TAG=${1:-small}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${TAG}_build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_small.py tests/test_gpu_fullsize.py -x -q --timeout 300 -k "small or bench" > gpurun_out/${TAG}_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/${TAG}_pytest.log
for n in 3 6; do
  timeout 300 python bench.py --n $n --no-cpu-baseline > gpurun_out/${TAG}_n$n.log 2>&1
  MP_SMALL_PROFILE=1 timeout 300 python bench.py --n $n --no-cpu-baseline --steps 2 --warmup 1 > gpurun_out/${TAG}_n${n}_prof.log 2>&1
done
