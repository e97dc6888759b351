# the GPU test suite on the bounds-checked debug build (-DMP_DEBUG_CHECKS=1), loaded through
# MP_LIB_PATH; compute-sanitizer is closed on this pool (profiles/r2/sanitizer_refused.log)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TAG=${1:-dbg}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${TAG}_build.log 2>&1
python bench_tools/build_variants.py debug=-DMP_DEBUG_CHECKS=1 >> gpurun_out/${TAG}_build.log 2>&1
MP_LIB_PATH=bench_tools/variants/debug.so timeout 3000 python -m pytest tests -m gpu -q -k "not test_every_entry and not test_power_records" > gpurun_out/${TAG}_pytest_debug.log 2>&1; echo "rc=$?" >> gpurun_out/${TAG}_pytest_debug.log
MP_LIB_PATH=bench_tools/variants/debug.so timeout 900 python bench_tools/r2/sanitize_target.py > gpurun_out/${TAG}_target_debug.log 2>&1; echo "rc=$?" >> gpurun_out/${TAG}_target_debug.log
MP_LIB_PATH=bench_tools/variants/debug.so timeout 600 python bench.py --n 12 --steps 1 --warmup 0 --no-cpu-baseline > gpurun_out/${TAG}_bench_n12_debug.log 2>&1; echo "rc=$?" >> gpurun_out/${TAG}_bench_n12_debug.log
