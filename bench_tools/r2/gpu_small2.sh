cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TAG=${1:-sm}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${TAG}_build.log 2>&1
for n in 3 4 5 6; do MP_SMALL_PROFILE=1 timeout 300 python bench.py --n $n --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/${TAG}_bench_n$n.log 2>&1; done
timeout 600 python bench.py --n 12 --no-cpu-baseline > gpurun_out/${TAG}_bench_n12.log 2>&1
timeout 600 python -m pytest tests/test_gpu_small.py tests/test_gpu_parity.py -x -q -k "small or row_reuse or transfer or remainder" > gpurun_out/${TAG}_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/${TAG}_pytest.log
