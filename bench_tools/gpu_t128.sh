# k_stats_sym with 128-thread blocks (1024 columns) vs 256: stats per power and benches n = 10, 11
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
T=${1:-t128}
for n in 10 11 12; do timeout 300 python bench_tools/stats_timing.py $n t256_n$n >> gpurun_out/${T}_stats.log 2>&1; done
for n in 10 11; do timeout 300 python bench.py --n $n --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/${T}_t256_bench_n$n.log 2>&1; done
cp paper_2409_17688_b200/libminplus.so /tmp/lib_orig.so
cp bench_tools/variants/t128.so paper_2409_17688_b200/libminplus.so
for n in 10 11 12; do timeout 300 python bench_tools/stats_timing.py $n t128_n$n >> gpurun_out/${T}_stats.log 2>&1; done
for n in 10 11; do timeout 300 python bench.py --n $n --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/${T}_t128_bench_n$n.log 2>&1; done
timeout 900 python -m pytest tests -m gpu -q -k "sym or symmetry or periodic" > gpurun_out/${T}_t128_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_t128_pytest.log
cp /tmp/lib_orig.so paper_2409_17688_b200/libminplus.so
