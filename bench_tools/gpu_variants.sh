# bench n = 12 (and 11) with each library variant in bench_tools/variants/*.so swapped in
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TAG=${1:-v}
cp paper_2409_17688_b200/libminplus.so /tmp/lib_orig.so
for f in bench_tools/variants/*.so; do
  b=$(basename $f .so)
  cp $f paper_2409_17688_b200/libminplus.so
  for n in 11 12; do timeout 300 python bench.py --n $n --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/${TAG}_${b}_n$n.log 2>&1; done
done
cp /tmp/lib_orig.so paper_2409_17688_b200/libminplus.so
