# SpMM L2 policies: X rows evict_last (bulk-copy cache hint), C rows streamed (st.global.cs),
# CTA order by column bands; plus the new setup kernels (tests first)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TAG=${1:-l2}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${TAG}_build.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_fullsize.py tests/test_gpu_parity.py -x -q --timeout 300 > gpurun_out/${TAG}_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/${TAG}_pytest.log
python bench_tools/build_variants.py cs=-DMP_SP_CSTORE_CS=1 hint=-DMP_SP_XHINT=1 cshint=-DMP_SP_CSTORE_CS=1,-DMP_SP_XHINT=1 b1cshint=-DMP_SP_CSTORE_CS=1,-DMP_SP_XHINT=1,-DMP_SP_BAND=1 b2cshint=-DMP_SP_CSTORE_CS=1,-DMP_SP_XHINT=1,-DMP_SP_BAND=2 >> gpurun_out/${TAG}_build.log 2>&1
timeout 300 python bench.py --n 12 --no-cpu-baseline --steps 6 > gpurun_out/${TAG}_base.log 2>&1
for v in cs hint cshint b1cshint b2cshint; do
  MP_LIB_PATH=bench_tools/variants/$v.so timeout 300 python bench.py --n 12 --no-cpu-baseline --steps 6 > gpurun_out/${TAG}_$v.log 2>&1
done
MP_LIB_PATH=bench_tools/variants/b1cshint.so timeout 300 python bench.py --n 12 --no-cpu-baseline --steps 6 --spmm-width 512 > gpurun_out/${TAG}_b1cshint_w512.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches.csv python bench.py --n 12 --steps 1 --warmup 0 --no-cpu-baseline > gpurun_out/${TAG}_ncu2.log 2>&1
