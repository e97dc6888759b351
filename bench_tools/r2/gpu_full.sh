# full GPU suite + smoke + bench lines + n=12 launch list
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TAG=${1:-full}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${TAG}_build.log 2>&1
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/${TAG}_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/${TAG}_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/${TAG}_smoke.log
for n in 12 11 10 9 6 3; do timeout 600 python bench.py --n $n --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/${TAG}_bench_n$n.log 2>&1; done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches_n12.csv python bench.py --n 12 --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/${TAG}_ncu_launch.log 2>&1
