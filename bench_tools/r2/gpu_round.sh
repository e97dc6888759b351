# full GPU suite, sanitizers on the small target, ncu of the small-N kernel and of k_spmm at n=12
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TAG=${1:-r2c}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${TAG}_build.log 2>&1
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/${TAG}_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/${TAG}_pytest.log
for tool in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool --error-exitcode 9 python bench_tools/r2/sanitize_target.py > gpurun_out/${TAG}_san_$tool.log 2>&1; echo "rc=$?" >> gpurun_out/${TAG}_san_$tool.log
done
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_small_run -c 2 -o gpurun_out/${TAG}_small_n6 -f python bench.py --n 6 --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/${TAG}_ncu_small.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_spmm -s 20 -c 1 -o gpurun_out/${TAG}_kspmm_n12 -f python bench.py --n 12 --steps 1 --warmup 0 --no-cpu-baseline > gpurun_out/${TAG}_ncu_spmm.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches_n12.csv python bench.py --n 12 --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/${TAG}_ncu_launch.log 2>&1
