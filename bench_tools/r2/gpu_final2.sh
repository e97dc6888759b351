# final evidence with the last code: GPU suite, smoke, bench lines, the fold product's DRAM
# traffic, the n = 12 launch list, ncu captures of k_fold and k_spmm
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TAG=${1:-f2}
bash bench_tools/r2/gpu_final.sh $TAG
timeout 1500 python -m pytest tests -m gpu -q --timeout 600 > gpurun_out/${TAG}_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/${TAG}_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/${TAG}_smoke.log
for n in 3 6; do timeout 300 python bench.py --n $n --no-cpu-baseline > gpurun_out/${TAG}_bench_n$n.log 2>&1; done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches_n12.csv python bench.py --n 12 --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/${TAG}_ncu_launch.log 2>&1
for k in k_spmm:40 k_fold:400; do
  name=${k%%:*}; skip=${k##*:}
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:$name -s $skip -c 1 -o gpurun_out/${TAG}_${name}_n12 -f python bench.py --n 12 --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/${TAG}_ncu_$name.log 2>&1
done
