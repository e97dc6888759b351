# order of the rows inside each fold level (MP_FOLD_ORDER q / p / s): reuse tests, bench n = 12, 11
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TAG=${1:-fo}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${TAG}_build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "reuse or fold_bytes" > gpurun_out/${TAG}_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/${TAG}_pytest.log
for n in 12 11; do for o in q p s; do
  MP_FOLD_ORDER=$o timeout 300 python bench.py --n $n --steps 5 --warmup 3 --no-cpu-baseline 2>&1 | grep '^{' | python -c "import json,sys; d=json.loads(sys.stdin.read()); b=d['breakdown_ms_per_step']; print('$o', $n, round(d['ms_per_step'],2), 'folds', round(b['folds'],2), 'spmm', round(b['product_kernel'],2))" >> gpurun_out/${TAG}_ab.log 2>&1
done; done
