# variants on the 1024-column SpMM: product time + bench n = 12; ncu capture of the default
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TAG=${1:-pp2}
cp paper_2409_17688_b200/libminplus.so /tmp/lib_orig.so
for f in bench_tools/variants/*.so; do
  b=$(basename $f .so)
  cp $f paper_2409_17688_b200/libminplus.so
  timeout 300 python bench_tools/product_timing.py 12 $b >> gpurun_out/${TAG}_ptime.log 2>&1
  timeout 300 python bench.py --n 12 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/${TAG}_${b}_n12.log 2>&1
done
cp /tmp/lib_orig.so paper_2409_17688_b200/libminplus.so
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_spmm -s 6 -c 1 -o gpurun_out/${TAG}_kspmm_default python bench_tools/product_timing.py 12 def > gpurun_out/${TAG}_ncu.log 2>&1
