# 128-thread k_stats_sym blocks as the default: GPU suite, smoke, benches
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
T=${1:-t128b}
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/${T}_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_pytest.log
timeout 300 python __graft_entry__.py smoke > gpurun_out/${T}_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_smoke.log
for n in 3 6 9 10 11; do timeout 300 python bench.py --n $n --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/${T}_bench_n$n.log 2>&1; done
timeout 900 python bench.py > gpurun_out/${T}_bench_default.log 2>&1
