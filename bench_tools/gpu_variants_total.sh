# bench n = 12 (total seconds to gamma_2, setup included) for each library variant
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TAG=${1:-vt}
cp paper_2409_17688_b200/libminplus.so /tmp/lib_orig.so
for f in bench_tools/variants/*.so; do
  b=$(basename $f .so)
  cp $f paper_2409_17688_b200/libminplus.so
  timeout 300 python bench.py --n 12 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/${TAG}_${b}_n12.log 2>&1
done
cp /tmp/lib_orig.so paper_2409_17688_b200/libminplus.so
