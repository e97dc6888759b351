cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/w37_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/w37_pytest.log
bash bench_tools/gpu_ptime.sh w37
for n in 10 11 12; do timeout 300 python bench.py --n $n --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/w37_bench_n$n.log 2>&1; done
