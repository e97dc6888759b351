# automatic width with 256-column CTAs for n <= 9: full GPU suite, benches n = 3..10 and default
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
T=${1:-w256b}
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/${T}_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_pytest.log
timeout 300 python __graft_entry__.py smoke > gpurun_out/${T}_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_smoke.log
for n in 3 6 9 10; do timeout 300 python bench.py --n $n --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/${T}_bench_n$n.log 2>&1; done
timeout 900 python bench.py > gpurun_out/${T}_bench_default.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_bench_default.log
