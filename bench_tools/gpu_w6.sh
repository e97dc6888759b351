cd $GRAFT_REPO_ROOT
TAG=${1:-w6}
mkdir -p gpurun_out
python bench_tools/setup_profile.py 12 > gpurun_out/${TAG}_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_tile_greedy|k_check_a" -c 2 -o gpurun_out/${TAG}_greedy python bench_tools/setup_profile.py 12 > gpurun_out/${TAG}_ncu.log 2>&1
