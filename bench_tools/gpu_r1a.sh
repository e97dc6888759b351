cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r1_gpuinfo.txt
timeout 300 python __graft_entry__.py smoke > gpurun_out/r1_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/r1_smoke.log
timeout 900 python -m pytest tests -m gpu -x -q -k "not large_n" > gpurun_out/r1_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r1_pytest.log
timeout 300 python bench.py --n 9 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r1_bench_n9.log 2>&1; echo "rc=$?" >> gpurun_out/r1_bench_n9.log
timeout 600 python bench.py --n 12 --steps 1 --warmup 1 --e2e-steps 1 --cpu-seconds 5 > gpurun_out/r1_bench_n12.log 2>&1; echo "rc=$?" >> gpurun_out/r1_bench_n12.log
