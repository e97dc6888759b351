# ncu evidence for round 1: launch list of the bench command (n=12) and one full capture of
# the product kernel at n=12 and n=9.  Each ncu run follows the same command run plainly.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
CMD="python bench.py --n 12 --steps 1 --warmup 1 --e2e-steps 1 --no-cpu-baseline"
$CMD > gpurun_out/r1_plain_n12.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r1_launches_n12.csv $CMD > gpurun_out/r1_ncu_launch_n12.log 2>&1
echo "launch list rc=$?" >> gpurun_out/r1_ncu_launch_n12.log
$CMD > gpurun_out/r1_plain_n12b.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_minplus -s 2 -c 1 -o gpurun_out/r1_kminplus_n12 $CMD > gpurun_out/r1_ncu_full_n12.log 2>&1
echo "full n12 rc=$?" >> gpurun_out/r1_ncu_full_n12.log
CMD9="python bench.py --n 9 --steps 1 --warmup 1 --e2e-steps 1 --no-cpu-baseline"
$CMD9 > gpurun_out/r1_plain_n9.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_minplus -s 30 -c 1 -o gpurun_out/r1_kminplus_n9 $CMD9 > gpurun_out/r1_ncu_full_n9.log 2>&1
echo "full n9 rc=$?" >> gpurun_out/r1_ncu_full_n9.log
