# A/B of compile-time variants at n = 12 (and n = 11): usage
#   gpurun -- 'bash bench_tools/r2/gpu_ab.sh TAG name=-DFLAG=1,-DOTHER=2 name2=-D...'
# builds the product library, then each variant into bench_tools/variants/<name>.so (loaded
# through MP_LIB_PATH; the product .so is never overwritten), and runs bench.py on each.
# The round-2 experiments recorded in DESIGN.md (SpMM CTA order MP_SP_BAND, grouping window
# MP_GRP_WIN, transfer-check width MP_XF_U, ...) ran this way; env switches (MP_LOOKAHEAD=2,
# MP_FP_TC=0) need no variant: set them on the bench command instead.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TAG=${1:-ab}
shift
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${TAG}_build.log 2>&1
[ $# -gt 0 ] && python bench_tools/build_variants.py "$@" >> gpurun_out/${TAG}_build.log 2>&1
for n in 12 11; do
  timeout 300 python bench.py --n $n --no-cpu-baseline > gpurun_out/${TAG}_n${n}_base.log 2>&1
  for spec in "$@"; do
    v=${spec%%=*}
    MP_LIB_PATH=bench_tools/variants/$v.so timeout 300 python bench.py --n $n --no-cpu-baseline > gpurun_out/${TAG}_n${n}_$v.log 2>&1
  done
done
