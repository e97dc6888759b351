# A/B: SpMM CTA order (column bands) and CTA width at n = 12 with the row-inclusion reuse
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TAG=${1:-band}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${TAG}_build.log 2>&1
python bench_tools/build_variants.py band1=-DMP_SP_BAND=1 band2=-DMP_SP_BAND=2 band4=-DMP_SP_BAND=4 band8=-DMP_SP_BAND=8 >> gpurun_out/${TAG}_build.log 2>&1
timeout 300 python bench.py --n 12 --no-cpu-baseline --steps 6 > gpurun_out/${TAG}_base.log 2>&1
for w in 512 256; do timeout 300 python bench.py --n 12 --no-cpu-baseline --steps 6 --spmm-width $w > gpurun_out/${TAG}_w$w.log 2>&1; done
for v in band1 band2 band4 band8; do
  MP_LIB_PATH=bench_tools/variants/$v.so timeout 300 python bench.py --n 12 --no-cpu-baseline --steps 6 > gpurun_out/${TAG}_$v.log 2>&1
  MP_LIB_PATH=bench_tools/variants/$v.so timeout 300 python bench.py --n 12 --no-cpu-baseline --steps 6 --spmm-width 512 > gpurun_out/${TAG}_${v}_w512.log 2>&1
done
