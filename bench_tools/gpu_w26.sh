cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python bench_tools/mul_bench.py > gpurun_out/w26_mul_bench.jsonl 2>&1
timeout 600 python bench_tools/mul_bench.py 52929 >> gpurun_out/w26_mul_bench.jsonl 2>&1
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/w26_bench.log 2>&1
