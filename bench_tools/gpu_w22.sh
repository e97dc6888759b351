cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
MP_TRACE=1 python bench_tools/setup_repeat.py 12 4 > gpurun_out/w22_trace.log 2>&1
