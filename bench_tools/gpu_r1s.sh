cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_sharded.py -q -x -k "not large_n and not n13" > gpurun_out/r1s_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r1s_pytest.log
for n in 3 6 9 11 12; do timeout 300 python bench.py --n $n --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 2 > gpurun_out/r1s_bench_n$n.log 2>&1; done
timeout 1500 python -m pytest tests -q -x -m gpu -k "large_n or small_cycles or n13" > gpurun_out/r1s_pytest_large.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r1s_pytest_large.log
CMD="python bench.py --n 12 --steps 1 --warmup 1 --e2e-steps 1 --no-cpu-baseline"
$CMD > gpurun_out/r1s_plain_n12.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_spmm -s 3 -c 1 -o gpurun_out/r1s_kspmm_n12 $CMD > gpurun_out/r1s_ncu_n12.log 2>&1
