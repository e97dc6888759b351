# programmatic dependent launches of the fold levels (MP_FOLD_PDL=0: plain launches): reuse and
# full-size record tests, bench n = 12, 11, 10 both ways
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TAG=${1:-pdl}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${TAG}_build.log 2>&1
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -x -q --timeout 600 -k "reuse or records or fold_bytes" > gpurun_out/${TAG}_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/${TAG}_pytest.log
for n in 12 11 10; do for v in 1 0 1 0; do
  MP_FOLD_PDL=$v timeout 300 python bench.py --n $n --steps 5 --warmup 3 --no-cpu-baseline 2>&1 | grep '^{' | python -c "import json,sys; d=json.loads(sys.stdin.read()); b=d['breakdown_ms_per_step']; print('pdl=$v', $n, round(d['ms_per_step'],3), 'folds', round(b['folds'],3))" >> gpurun_out/${TAG}_ab.log 2>&1
done; done
