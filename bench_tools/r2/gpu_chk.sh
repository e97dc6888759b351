# vectorised transfer-hint check + grid-wide cheap statistics: tests and bench
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TAG=${1:-chk}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${TAG}_build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q --timeout 300 -k "transfer" > gpurun_out/${TAG}_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/${TAG}_pytest.log
timeout 900 python -m pytest tests/test_gpu_fullsize.py -x -q --timeout 300 -k "bench" >> gpurun_out/${TAG}_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/${TAG}_pytest.log
for n in 12 11 10; do
  timeout 300 python bench.py --n $n --no-cpu-baseline --steps 6 > gpurun_out/${TAG}_n$n.log 2>&1
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches.csv python bench.py --n 12 --steps 1 --warmup 0 --no-cpu-baseline > gpurun_out/${TAG}_ncu2.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_check_xfer -c 1 -o gpurun_out/${TAG}_kxfer -f python bench.py --n 12 --steps 1 --warmup 0 --no-cpu-baseline > gpurun_out/${TAG}_ncu.log 2>&1
