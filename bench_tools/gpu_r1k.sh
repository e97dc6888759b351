cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_sharded.py -q -x -k "not large_n and not n13" > gpurun_out/r1k_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r1k_pytest.log
timeout 300 python bench.py --n 12 --steps 3 --warmup 3 --e2e-steps 1 --cpu-seconds 10 > gpurun_out/r1k_bench_n12.log 2>&1
CMD="python bench.py --n 12 --steps 1 --warmup 1 --e2e-steps 1 --no-cpu-baseline"
$CMD > gpurun_out/r1k_plain_n12.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_spmm -s 3 -c 1 -o gpurun_out/r1k_kspmm_n12 $CMD > gpurun_out/r1k_ncu_n12.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r1k_launches_n12.csv $CMD > gpurun_out/r1k_ncu_launch.log 2>&1
echo "ncu rc=$?" >> gpurun_out/r1k_ncu_n12.log
