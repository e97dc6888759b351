cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r1f_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r1f_pytest.log
timeout 1500 python bench_tools/n13.py 13 > gpurun_out/r1f_n13.log 2>&1; echo "rc=$?" >> gpurun_out/r1f_n13.log
CMD="python bench.py --n 12 --steps 1 --warmup 1 --e2e-steps 1 --no-cpu-baseline --kernel spmm"
$CMD > gpurun_out/r1f_plain_n12.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_spmm -s 3 -c 1 -o gpurun_out/r1f_kspmm_n12 $CMD > gpurun_out/r1f_ncu_n12.log 2>&1
echo "ncu rc=$?" >> gpurun_out/r1f_ncu_n12.log
