cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
MP_TRACE=1 python bench_tools/setup_repeat.py 6 3 > gpurun_out/w32_trace6.log 2>&1
MP_TRACE=1 python bench_tools/setup_repeat.py 3 3 > gpurun_out/w32_trace3.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/w32_launches6.csv python bench_tools/setup_repeat.py 6 2 > gpurun_out/w32_ncu6.log 2>&1
