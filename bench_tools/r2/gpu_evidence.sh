# round-2 evidence run: GPU suite (n = 10/11/12 golden records incl. SHA-256 of every power),
# smoke, bench lines (default with the CPU oracle beside it), reference arm, n = 13, the
# streamed element-wise n = 11 compare, launch list, ncu captures of the step's kernels
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TAG=${1:-ev}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${TAG}_build.log 2>&1
timeout 2400 python -m pytest tests -m gpu -q --timeout 900 > gpurun_out/${TAG}_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/${TAG}_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/${TAG}_smoke.log
timeout 900 python bench.py > gpurun_out/${TAG}_bench_default.log 2>&1
for n in 3 6 9 10 11; do timeout 600 python bench.py --n $n --no-cpu-baseline > gpurun_out/${TAG}_bench_n$n.log 2>&1; done
timeout 600 python bench.py --n 12 --no-cpu-baseline --no-row-reuse > gpurun_out/${TAG}_bench_n12_noreuse.log 2>&1
timeout 900 python bench.py --n 13 --no-cpu-baseline --steps 3 --warmup 1 > gpurun_out/${TAG}_bench_n13.log 2>&1
timeout 900 python bench.py --impl reference > gpurun_out/${TAG}_bench_reference.log 2>&1
timeout 900 python bench_tools/n13.py 13 > gpurun_out/${TAG}_n13.log 2>&1
MP_FULL_PARITY=1 timeout 1800 python -m pytest tests/test_gpu_fullsize.py -q -s -k streamed > gpurun_out/${TAG}_streamed_n11.log 2>&1; echo "rc=$?" >> gpurun_out/${TAG}_streamed_n11.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches_n12.csv python bench.py --n 12 --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/${TAG}_ncu_launch.log 2>&1
# one --set full capture per kernel of the n = 12 step (-s skips the warm-up run's launches)
for k in k_spmm:40 k_fold:400 k_fp_tc:40 k_check_xfer:1 k_stats_sym:40; do
  name=${k%%:*}; skip=${k##*:}
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:$name -s $skip -c 1 -o gpurun_out/${TAG}_${name}_n12 -f python bench.py --n 12 --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/${TAG}_ncu_$name.log 2>&1
done
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_small_run -s 3 -c 1 -o gpurun_out/${TAG}_small_n3 -f python bench.py --n 3 --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/${TAG}_ncu_small.log 2>&1
