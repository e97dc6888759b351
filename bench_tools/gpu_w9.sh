cd $GRAFT_REPO_ROOT
TAG=${1:-w9}
mkdir -p gpurun_out
python bench_tools/setup_profile.py 12 > gpurun_out/${TAG}_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_spmm" -s 3 -c 1 -o gpurun_out/${TAG}_spmm python bench_tools/setup_profile.py 12 > gpurun_out/${TAG}_ncu.log 2>&1
