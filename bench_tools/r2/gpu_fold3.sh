cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TAG=${1:-fold3}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${TAG}_build.log 2>&1
python bench_tools/build_variants.py rowmaj=-DMP_SP_FOLD_COLMAJOR=0 >> gpurun_out/${TAG}_build.log 2>&1
for n in 12 10; do
  MP_LIB_PATH=bench_tools/variants/rowmaj.so timeout 300 python bench.py --n $n --no-cpu-baseline --steps 6 > gpurun_out/${TAG}_n${n}_rowmaj.log 2>&1
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches_n10.csv python bench.py --n 10 --steps 1 --warmup 0 --no-cpu-baseline > gpurun_out/${TAG}_ncu2.log 2>&1
MP_FOLD_SPMM=0 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches_n10_sep.csv python bench.py --n 10 --steps 1 --warmup 0 --no-cpu-baseline > gpurun_out/${TAG}_ncu3.log 2>&1
