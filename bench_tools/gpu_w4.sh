cd $GRAFT_REPO_ROOT
TAG=${1:-w4}
mkdir -p gpurun_out
MP_TRACE=1 python bench_tools/setup_profile.py 12 > gpurun_out/${TAG}_trace.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:"k_support|k_row_popc|k_bits|k_tile|k_scan|k_group_masks|k_tile_bal|k_x1|k_chunk|k_iota|k_make|k_encode|k_check" --log-file gpurun_out/${TAG}_setup_launches.csv python bench_tools/setup_profile.py 12 > gpurun_out/${TAG}_ncu.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/${TAG}_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/${TAG}_pytest.log
for n in 10 11 12; do timeout 300 python bench.py --n $n --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/${TAG}_bench_n$n.log 2>&1; done
