cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TAG=${1:-fs}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${TAG}_build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_fullsize.py -x -q -k "foldstats or nolookahead or bench" > gpurun_out/${TAG}_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/${TAG}_pytest.log
for v in 0 1; do
  MP_FOLD_STATS=$v timeout 600 python bench.py --n 12 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/${TAG}_bench_n12_fs$v.log 2>&1
  MP_FOLD_STATS=$v timeout 600 python bench.py --n 11 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/${TAG}_bench_n11_fs$v.log 2>&1
done
MP_LOOKAHEAD=0 timeout 600 python bench.py --n 12 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/${TAG}_bench_n12_nola.log 2>&1
