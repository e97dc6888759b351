# quick check of a kernel change: GPU parity tests + n = 10..12 benches (no CPU baseline)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TAG=${1:-q}
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/${TAG}_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/${TAG}_pytest.log
for n in 10 11 12; do timeout 300 python bench.py --n $n --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/${TAG}_bench_n$n.log 2>&1; done
