cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "not large_n and not n13" > gpurun_out/r1j_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r1j_pytest.log
for st in 2 3; do MP_SPMM_STAGES=$st timeout 300 python bench.py --n 12 --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 1 --kernel spmm > gpurun_out/r1j_bench_n12_st$st.log 2>&1; done
MP_SPMM_STAGES=2 timeout 300 python bench.py --n 11 --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 1 --kernel spmm > gpurun_out/r1j_bench_n11_st2.log 2>&1
MP_SPMM_STAGES=2 timeout 1200 python -m pytest tests -q -x -m gpu -k "large_n or sharded" > gpurun_out/r1j_pytest_large.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r1j_pytest_large.log
