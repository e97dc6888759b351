cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TAG=${1:-tc3}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${TAG}_build.log 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q --timeout 300 > gpurun_out/${TAG}_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/${TAG}_pytest.log
for n in 12 11 10; do
  timeout 300 python bench.py --n $n --no-cpu-baseline > gpurun_out/${TAG}_bench_n$n.log 2>&1
done
