cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r1c_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r1c_pytest.log
for n in 3 6 9; do timeout 300 python bench.py --n $n --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r1c_bench_n$n.log 2>&1; done
timeout 900 python bench.py > gpurun_out/r1c_bench_default.log 2>&1; echo "rc=$?" >> gpurun_out/r1c_bench_default.log
