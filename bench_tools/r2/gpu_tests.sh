# full GPU test suite
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TAG=${1:-tests}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${TAG}_build.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q --timeout 600 ${PYTEST_K:+-k "$PYTEST_K"} > gpurun_out/${TAG}_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/${TAG}_pytest.log
