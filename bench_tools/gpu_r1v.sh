cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/r1v_bench_default.log 2>&1; echo "rc=$?" >> gpurun_out/r1v_bench_default.log
timeout 600 python bench.py --impl reference > gpurun_out/r1v_bench_reference.log 2>&1; echo "rc=$?" >> gpurun_out/r1v_bench_reference.log
timeout 300 python __graft_entry__.py smoke > gpurun_out/r1v_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/r1v_smoke.log
for n in 3 6 9 10 11; do timeout 300 python bench.py --n $n --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r1v_bench_n$n.log 2>&1; done
timeout 300 python bench.py --n 12 --steps 2 --warmup 3 --no-cpu-baseline --kernel tiles > gpurun_out/r1v_bench_n12_tiles.log 2>&1
CMD="python bench.py --n 12 --steps 1 --warmup 1 --e2e-steps 1 --no-cpu-baseline"
$CMD > gpurun_out/r1v_plain_n12.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r1v_launches_n12.csv $CMD > gpurun_out/r1v_ncu_launch.log 2>&1
