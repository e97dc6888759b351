# k_fold_wave (one persistent fold launch) against the per-level k_fold launches (MP_FOLD=levels):
# reuse parity tests, then bench.py at n = 12, 11, 10 both ways
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TAG=${1:-wave}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${TAG}_build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -x -q --timeout 300 -k "reuse or bench" > gpurun_out/${TAG}_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/${TAG}_pytest.log
for n in 12 11 10; do
  timeout 300 python bench.py --n $n --no-cpu-baseline > gpurun_out/${TAG}_n${n}.log 2>&1
  MP_FOLD=levels timeout 300 python bench.py --n $n --no-cpu-baseline > gpurun_out/${TAG}_n${n}_levels.log 2>&1
done
