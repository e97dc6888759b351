# 256-column SpMM CTAs: product time per width at n = 9, 10, 11; width parity tests
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TAG=${1:-w256}
for n in 9 10 11; do for W in 256 512 1024; do
  MP_WIDTH=$W timeout 300 python bench_tools/product_timing.py $n W$W >> gpurun_out/${TAG}_ptime.log 2>&1
done; done
timeout 900 python -m pytest tests -m gpu -q -k "width" > gpurun_out/${TAG}_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/${TAG}_pytest.log
