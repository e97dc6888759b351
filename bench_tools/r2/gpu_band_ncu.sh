# ncu of k_spmm with column-block-major CTA order (MP_SP_BAND=1) vs the default
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TAG=${1:-bandncu}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${TAG}_build.log 2>&1
python bench_tools/build_variants.py band1=-DMP_SP_BAND=1 band4=-DMP_SP_BAND=4 >> gpurun_out/${TAG}_build.log 2>&1
for v in band1 band4; do
MP_LIB_PATH=bench_tools/variants/$v.so timeout 900 ncu --set full --clock-control none -k regex:k_spmm -s 40 -c 1 -o gpurun_out/${TAG}_$v -f python bench.py --n 12 --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/${TAG}_ncu_$v.log 2>&1
done
