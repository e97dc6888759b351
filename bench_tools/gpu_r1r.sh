cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python bench_tools/small_n_timing.py 3 6 9 11 > gpurun_out/r1r_small_n.log 2>&1
