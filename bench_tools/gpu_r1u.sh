cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_sharded.py -q -x -k "not large_n and not n13" > gpurun_out/r1u_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r1u_pytest.log
for n in 9 11 12; do timeout 300 python bench.py --n $n --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 2 > gpurun_out/r1u_bench_n$n.log 2>&1; done
timeout 1500 python -m pytest tests -q -x -m gpu -k "large_n or small_cycles or n13" > gpurun_out/r1u_pytest_large.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r1u_pytest_large.log
timeout 600 python bench_tools/n13.py 13 > gpurun_out/r1u_n13.log 2>&1
