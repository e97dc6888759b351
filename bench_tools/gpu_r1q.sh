cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
MP_TRACE=1 timeout 300 python bench.py --n 12 --steps 2 --warmup 1 --no-cpu-baseline --e2e-steps 1 > gpurun_out/r1q_trace_n12.log 2>&1
MP_TRACE=1 timeout 300 python bench.py --n 9 --steps 2 --warmup 1 --no-cpu-baseline --e2e-steps 1 > gpurun_out/r1q_trace_n9.log 2>&1
for n in 9 12; do timeout 300 python bench.py --n $n --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 2 > gpurun_out/r1q_bench_n$n.log 2>&1; done
