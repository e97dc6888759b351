# product_timing.py for each library variant in bench_tools/variants/*.so
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TAG=${1:-pt}
cp paper_2409_17688_b200/libminplus.so /tmp/lib_orig.so
for f in bench_tools/variants/*.so; do
  b=$(basename $f .so)
  cp $f paper_2409_17688_b200/libminplus.so
  timeout 300 python bench_tools/stats_timing.py 12 $b >> gpurun_out/${TAG}_ptime.log 2>&1
done
cp /tmp/lib_orig.so paper_2409_17688_b200/libminplus.so
