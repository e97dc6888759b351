# row-reuse check: targeted tests, then n=12 with and without the reuse
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TAG=${1:-dag}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${TAG}_build.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_parity.py -x -q -k "row_reuse or words_source or transfer" > gpurun_out/${TAG}_pytest_dag.log 2>&1; echo "rc=$?" >> gpurun_out/${TAG}_pytest_dag.log
timeout 1200 python -m pytest tests/test_gpu_fullsize.py tests/test_gpu_small.py -x -q > gpurun_out/${TAG}_pytest_full.log 2>&1; echo "rc=$?" >> gpurun_out/${TAG}_pytest_full.log
for n in 12 11 10; do
  timeout 600 python bench.py --n $n --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/${TAG}_bench_n$n.log 2>&1
done
timeout 600 python bench.py --n 12 --steps 3 --warmup 3 --no-cpu-baseline --no-row-reuse > gpurun_out/${TAG}_bench_n12_noreuse.log 2>&1
for n in 3 6; do timeout 600 python bench.py --n $n --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/${TAG}_bench_n$n.log 2>&1; done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches_n12.csv python bench.py --n 12 --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/${TAG}_ncu_launch.log 2>&1
