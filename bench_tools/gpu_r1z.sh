# full GPU suite on the default build, benches for every config, product-time variants
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TAG=${1:-r1z}
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/${TAG}_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/${TAG}_pytest.log
for n in 3 6 9 10 11; do timeout 300 python bench.py --n $n --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/${TAG}_bench_n$n.log 2>&1; done
bash bench_tools/gpu_ptime.sh ${TAG}
cp paper_2409_17688_b200/libminplus.so /tmp/lib_orig.so
cp bench_tools/variants/k_ppl8.so paper_2409_17688_b200/libminplus.so
for n in 6 9 10; do timeout 300 python bench.py --n $n --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/${TAG}_ppl8_bench_n$n.log 2>&1; done
cp /tmp/lib_orig.so paper_2409_17688_b200/libminplus.so
