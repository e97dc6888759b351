cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
CMD="python bench.py --n 12 --steps 1 --warmup 1 --e2e-steps 1 --no-cpu-baseline"
$CMD > gpurun_out/r1m_plain_n12.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_spmm -s 3 -c 1 -o gpurun_out/r1m_kspmm_n12 $CMD > gpurun_out/r1m_ncu_n12.log 2>&1
echo "ncu rc=$?" >> gpurun_out/r1m_ncu_n12.log
