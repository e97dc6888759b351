# transfer-check variants (256 / 512 columns per lane) at n = 12; transfer tests
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TAG=${1:-xf}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${TAG}_build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -x -q --timeout 300 -k "transfer or bench" > gpurun_out/${TAG}_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/${TAG}_pytest.log
python bench_tools/build_variants.py u2=-DMP_XF_U=2 >> gpurun_out/${TAG}_build.log 2>&1
timeout 300 python bench.py --n 12 --no-cpu-baseline > gpurun_out/${TAG}_n12.log 2>&1
MP_LIB_PATH=bench_tools/variants/u2.so timeout 300 python bench.py --n 12 --no-cpu-baseline > gpurun_out/${TAG}_n12_u2.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches.csv python bench.py --n 12 --steps 1 --warmup 0 --no-cpu-baseline > gpurun_out/${TAG}_ncu2.log 2>&1
