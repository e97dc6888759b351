cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TAG=${1:-tc}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${TAG}_build.log 2>&1
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/${TAG}_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/${TAG}_pytest.log
for n in 12 11 10 9; do
  timeout 600 python bench.py --n $n --no-cpu-baseline > gpurun_out/${TAG}_bench_n$n.log 2>&1
done
MP_FP_TC=0 timeout 600 python bench.py --n 12 --no-cpu-baseline > gpurun_out/${TAG}_bench_n12_notc.log 2>&1
for n in 3 6; do timeout 300 python bench.py --n $n --no-cpu-baseline > gpurun_out/${TAG}_bench_n$n.log 2>&1; done
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_fp_tc -s 10 -c 1 -o gpurun_out/${TAG}_kfptc -f python bench.py --n 12 --steps 1 --warmup 0 --no-cpu-baseline > gpurun_out/${TAG}_ncu.log 2>&1
