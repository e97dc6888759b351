# GPU parity tests on the default build, then the n = 11/12 benches of each variant
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TAG=${1:-tv}
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/${TAG}_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/${TAG}_pytest.log
bash bench_tools/gpu_variants.sh ${TAG}
