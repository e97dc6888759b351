# n = 12 bench line, then one ncu --set full capture each of k_spmm, k_fold and k_stats_sym
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TAG=${1:-ncu12}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${TAG}_build.log 2>&1
timeout 600 python bench.py --n 12 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/${TAG}_bench_n12.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_spmm -s 10 -c 1 -o gpurun_out/${TAG}_kspmm -f python bench.py --n 12 --steps 1 --warmup 0 --no-cpu-baseline > gpurun_out/${TAG}_ncu1.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_fold -s 60 -c 1 -o gpurun_out/${TAG}_kfold -f python bench.py --n 12 --steps 1 --warmup 0 --no-cpu-baseline > gpurun_out/${TAG}_ncu2.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_stats_sym -s 10 -c 1 -o gpurun_out/${TAG}_kstats -f python bench.py --n 12 --steps 1 --warmup 0 --no-cpu-baseline > gpurun_out/${TAG}_ncu3.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_check_a -c 1 -o gpurun_out/${TAG}_kcheck -f python bench.py --n 12 --steps 1 --warmup 0 --no-cpu-baseline > gpurun_out/${TAG}_ncu4.log 2>&1
