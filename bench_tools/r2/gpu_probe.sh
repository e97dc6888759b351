# quick probes: n=13 record time, k_check_a and a large k_fold level under ncu
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TAG=${1:-probe}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${TAG}_build.log 2>&1
timeout 900 python bench_tools/n13.py 13 > gpurun_out/${TAG}_n13.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_check_a -c 1 -o gpurun_out/${TAG}_kcheck -f python bench.py --n 12 --steps 1 --warmup 0 --no-cpu-baseline > gpurun_out/${TAG}_ncu4.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_fold -s 4 -c 1 -o gpurun_out/${TAG}_kfold -f python bench.py --n 12 --steps 1 --warmup 0 --no-cpu-baseline > gpurun_out/${TAG}_ncu2.log 2>&1
