# k_fold_wave (one persistent fold launch) against the per-level k_fold launches (MP_FOLD=levels):
# reuse parity tests, then bench.py at n = 12 and 11 for the variants (blocks per SM as builds,
# diagonal spacing MP_WAVE_C and publish interval MP_WAVE_F as env switches)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TAG=${1:-wave}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${TAG}_build.log 2>&1
python bench_tools/build_variants.py minb2=-DMP_WAVE_MINB=2 minb4=-DMP_WAVE_MINB=4 >> gpurun_out/${TAG}_build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q --timeout 300 -k "reuse" > gpurun_out/${TAG}_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/${TAG}_pytest.log
b() { timeout 300 python bench.py --n $1 --steps 3 --warmup 3 --no-cpu-baseline 2>&1 | grep '^{' | python -c "import json,sys; d=json.loads(sys.stdin.read()); b=d['breakdown_ms_per_step']; print('$2', $1, round(d['ms_per_step'],2), 'folds', round(b['folds'],2), 'prod', round(b['product_kernel'],2))" >> gpurun_out/${TAG}_ab.log 2>&1; }
for n in 12 11; do
  MP_FOLD=levels b $n levels
  b $n c2f4
  MP_WAVE_C=1 b $n c1f4
  MP_WAVE_C=4 b $n c4f4
  MP_WAVE_F=1 b $n c2f1
  MP_WAVE_F=8 b $n c2f8
  MP_WAVE_F=16 MP_WAVE_C=4 b $n c4f16
  MP_LIB_PATH=bench_tools/variants/minb2.so b $n minb2
  MP_LIB_PATH=bench_tools/variants/minb4.so b $n minb4
done
