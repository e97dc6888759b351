# round-1 final measurement sweep (after the row grouping, 4-row-group SpMM, symmetry)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
T=${1:-r1w}
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/${T}_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_pytest.log
timeout 900 python bench.py > gpurun_out/${T}_bench_default.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_bench_default.log
timeout 600 python bench.py --impl reference > gpurun_out/${T}_bench_reference.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_bench_reference.log
timeout 300 python __graft_entry__.py smoke > gpurun_out/${T}_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_smoke.log
for n in 3 6 9 10 11; do timeout 300 python bench.py --n $n --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/${T}_bench_n$n.log 2>&1; done
timeout 300 python bench.py --n 12 --steps 3 --warmup 3 --no-cpu-baseline --no-symmetry > gpurun_out/${T}_bench_n12_nosym.log 2>&1
timeout 600 python bench.py --n 12 --steps 2 --warmup 3 --no-cpu-baseline --kernel tiles --no-symmetry > gpurun_out/${T}_bench_n12_tiles.log 2>&1
MP_TRACE=1 timeout 600 python bench_tools/n13.py 13 > gpurun_out/${T}_n13.log 2>&1
CMD="python bench.py --n 12 --steps 1 --warmup 1 --e2e-steps 1 --no-cpu-baseline"
$CMD > gpurun_out/${T}_plain_n12.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${T}_launches_n12.csv $CMD > gpurun_out/${T}_ncu_launch.log 2>&1
