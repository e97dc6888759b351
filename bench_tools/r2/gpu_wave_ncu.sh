# one ncu --set full capture of k_fold_wave (2 blocks per SM build) and of k_fold at n = 12
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TAG=${1:-wncu}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${TAG}_build.log 2>&1
python bench_tools/build_variants.py minb2=-DMP_WAVE_MINB=2 >> gpurun_out/${TAG}_build.log 2>&1
MP_LIB_PATH=bench_tools/variants/minb2.so timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_fold_wave -s 2 -c 1 -o gpurun_out/${TAG}_wave python bench.py --n 12 --steps 1 --warmup 0 --no-cpu-baseline > gpurun_out/${TAG}_wave.log 2>&1
MP_FOLD=levels timeout 600 ncu --set full --clock-control none -k regex:'k_fold$|k_fold[^_]' -s 40 -c 1 -o gpurun_out/${TAG}_levels python bench.py --n 12 --steps 1 --warmup 0 --no-cpu-baseline > gpurun_out/${TAG}_levels.log 2>&1
