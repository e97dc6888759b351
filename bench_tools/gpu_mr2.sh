# k_stats_sym rows-per-block floor (only while >= 1 block per SM): benches, then the GPU suite
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
T=${1:-mr2}
for n in 3 6 9 10 11; do timeout 300 python bench.py --n $n --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/${T}_bench_n$n.log 2>&1; done
for n in 3 6 9; do timeout 300 python bench.py --n $n --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/${T}_bench_n${n}_again.log 2>&1; done
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/${T}_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_pytest.log
timeout 900 python bench.py > gpurun_out/${T}_bench_default.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_bench_default.log
