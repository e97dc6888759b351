cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TAG=${1:-tv}
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "spmm or random or large" > gpurun_out/${TAG}_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/${TAG}_pytest.log
bash bench_tools/gpu_variants.sh ${TAG}
