# ring-shape variants (product time at n = 12 and bench), then the default bench again
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TAG=${1:-z3}
cp paper_2409_17688_b200/libminplus.so /tmp/lib_orig.so
for f in bench_tools/variants/*.so; do
  b=$(basename $f .so)
  cp $f paper_2409_17688_b200/libminplus.so
  timeout 300 python bench_tools/product_timing.py 12 $b >> gpurun_out/${TAG}_ptime.log 2>&1
  timeout 300 python bench_tools/product_timing.py 11 $b >> gpurun_out/${TAG}_ptime.log 2>&1
done
cp /tmp/lib_orig.so paper_2409_17688_b200/libminplus.so
timeout 900 python bench.py > gpurun_out/${TAG}_bench_default.log 2>&1; echo "rc=$?" >> gpurun_out/${TAG}_bench_default.log
