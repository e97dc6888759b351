# A/B: small-N kernel, k_stats_sym 8 vs 16 columns per thread, 64-row SpMM tiles (built on the box)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TAG=${1:-ab}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${TAG}_build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_small.py tests/test_gpu_fullsize.py -x -q -k "not streamed" > gpurun_out/${TAG}_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/${TAG}_pytest.log
for n in 3 6; do timeout 300 python bench.py --n $n --no-cpu-baseline > gpurun_out/${TAG}_bench_n$n.log 2>&1; done
for c in 8 16; do
  MP_STATS_COLS=$c timeout 600 python bench.py --n 12 --no-cpu-baseline > gpurun_out/${TAG}_bench_n12_st$c.log 2>&1
  MP_STATS_COLS=$c MP_LOOKAHEAD=0 timeout 600 python bench.py --n 12 --no-cpu-baseline > gpurun_out/${TAG}_bench_n12_st${c}_nola.log 2>&1
done
python bench_tools/build_variants.py r64c1s4=-DMP_SP_ROWS=64,-DMP_SP_CTAS=1,-DMP_SP_STAGES=4 r64c1s5=-DMP_SP_ROWS=64,-DMP_SP_CTAS=1,-DMP_SP_STAGES=5 >> gpurun_out/${TAG}_build.log 2>&1
for v in r64c1s4 r64c1s5; do
  MP_LIB_PATH=bench_tools/variants/$v.so timeout 600 python bench.py --n 12 --no-cpu-baseline > gpurun_out/${TAG}_bench_n12_$v.log 2>&1
done
