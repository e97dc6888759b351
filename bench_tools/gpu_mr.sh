# k_stats_sym rows per block floor: benches n = 6, 9, 10 per variant, then the GPU suite and benches
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
T=${1:-mr}
cp paper_2409_17688_b200/libminplus.so /tmp/lib_orig.so
for f in bench_tools/variants/mr*.so; do
  b=$(basename $f .so)
  cp $f paper_2409_17688_b200/libminplus.so
  for n in 6 9 10; do timeout 300 python bench.py --n $n --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/${T}_${b}_bench_n$n.log 2>&1; done
done
cp /tmp/lib_orig.so paper_2409_17688_b200/libminplus.so
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/${T}_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_pytest.log
for n in 3 6 9 10 11; do timeout 300 python bench.py --n $n --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/${T}_bench_n$n.log 2>&1; done
timeout 900 python bench.py > gpurun_out/${T}_bench_default.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_bench_default.log
