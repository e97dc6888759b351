# each library variant in bench_tools/variants/*.so: product time at n = 12, a parity subset, bench n = 12
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TAG=${1:-ppl}
cp paper_2409_17688_b200/libminplus.so /tmp/lib_orig.so
for f in bench_tools/variants/*.so; do
  b=$(basename $f .so)
  cp $f paper_2409_17688_b200/libminplus.so
  timeout 300 python bench_tools/product_timing.py 12 $b >> gpurun_out/${TAG}_ptime.log 2>&1
  timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "(transfer and spmm) or symmetry_power_rows_full or (large_n_sampled and 12)" > gpurun_out/${TAG}_${b}_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/${TAG}_${b}_pytest.log
  timeout 300 python bench.py --n 12 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/${TAG}_${b}_n12.log 2>&1
done
cp /tmp/lib_orig.so paper_2409_17688_b200/libminplus.so
