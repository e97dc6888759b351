# k_stats / k_stats_sym: fewer instructions per row (split 64-bit weights, tracked first keys);
# per-power times, GPU tests, default bench, ncu of k_stats_sym
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TAG=${1:-st4}
timeout 300 python bench_tools/stats_timing.py 12 d8 >> gpurun_out/${TAG}_stats.log 2>&1
cp paper_2409_17688_b200/libminplus.so /tmp/lib_orig.so
for f in bench_tools/variants/st_*.so; do
  b=$(basename $f .so)
  cp $f paper_2409_17688_b200/libminplus.so
  timeout 300 python bench_tools/stats_timing.py 12 $b >> gpurun_out/${TAG}_stats.log 2>&1
done
cp /tmp/lib_orig.so paper_2409_17688_b200/libminplus.so
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/${TAG}_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/${TAG}_pytest.log
timeout 600 python bench.py > gpurun_out/${TAG}_bench_default.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_stats_sym -s 5 -c 1 -o gpurun_out/${TAG}_kstats_sym python bench_tools/stats_timing.py 12 ncu > gpurun_out/${TAG}_ncu1.log 2>&1
