cd $GRAFT_REPO_ROOT
TAG=${1:-w21}
mkdir -p gpurun_out
MP_TRACE=1 timeout 600 python bench_tools/n13.py 13 > gpurun_out/${TAG}_n13.log 2>&1
python bench_tools/setup_profile.py 12 > gpurun_out/${TAG}_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_spmm" -s 3 -c 1 -o gpurun_out/${TAG}_spmm python bench_tools/setup_profile.py 12 > gpurun_out/${TAG}_ncu.log 2>&1
