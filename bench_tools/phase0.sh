set -x
cd $GRAFT_REPO_ROOT
nvidia-smi --query-gpu=index,name,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active --format=csv
nvidia-smi --query-gpu=index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap --format=csv -lms 200 > gpurun_out/phase0_clocks.csv &
SMI=$!
timeout 300 ./bench_tools/dpx_peak | tee gpurun_out/phase0_dpx.jsonl
kill $SMI
lscpu | head -20 > gpurun_out/phase0_lscpu.txt; nproc >> gpurun_out/phase0_lscpu.txt
