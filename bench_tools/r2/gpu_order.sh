# extras row order (default) against the windowed greedy tiles (MP_GROUP_ORDER=greedy): reuse
# parity tests, full-size golden records, bench.py at n = 12, 11, 10 both ways, ncu of k_spmm
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TAG=${1:-order}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${TAG}_build.log 2>&1
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -x -q --timeout 600 -k "reuse or records" > gpurun_out/${TAG}_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/${TAG}_pytest.log
for n in 12 11 10; do
  MP_TRACE=1 timeout 300 python bench.py --n $n --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/${TAG}_trace_n$n.log 2>&1
  timeout 300 python bench.py --n $n --no-cpu-baseline > gpurun_out/${TAG}_n$n.log 2>&1
  MP_GROUP_ORDER=greedy timeout 300 python bench.py --n $n --no-cpu-baseline > gpurun_out/${TAG}_n${n}_greedy.log 2>&1
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_spmm -s 3 -c 1 -o gpurun_out/${TAG}_kspmm python bench.py --n 12 --steps 1 --warmup 0 --no-cpu-baseline > gpurun_out/${TAG}_ncu.log 2>&1
