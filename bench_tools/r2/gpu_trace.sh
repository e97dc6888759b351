# phase trace of the n = 12 run (MP_TRACE=1), tests of the touched paths, bench
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TAG=${1:-trace}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${TAG}_build.log 2>&1
MP_TRACE=1 timeout 300 python bench.py --n 12 --no-cpu-baseline --steps 2 --warmup 1 > gpurun_out/${TAG}_n12_trace.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_fullsize.py tests/test_gpu_parity.py -x -q --timeout 300 > gpurun_out/${TAG}_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/${TAG}_pytest.log
for n in 12 11 10; do timeout 300 python bench.py --n $n --no-cpu-baseline > gpurun_out/${TAG}_n$n.log 2>&1; done
