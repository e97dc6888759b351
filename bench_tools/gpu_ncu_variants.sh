# one ncu --set full capture of k_spmm per library variant (product_timing.py, n = 12)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TAG=${1:-nv}
cp paper_2409_17688_b200/libminplus.so /tmp/lib_orig.so
for f in bench_tools/variants/*.so; do
  b=$(basename $f .so)
  cp $f paper_2409_17688_b200/libminplus.so
  timeout 300 python bench_tools/product_timing.py 12 $b > gpurun_out/${TAG}_${b}_plain.log 2>&1 && \
  timeout 600 ncu --set full --clock-control none -k regex:k_spmm -s 6 -c 1 -o gpurun_out/${TAG}_${b} python bench_tools/product_timing.py 12 $b > gpurun_out/${TAG}_${b}_ncu.log 2>&1
done
cp /tmp/lib_orig.so paper_2409_17688_b200/libminplus.so
