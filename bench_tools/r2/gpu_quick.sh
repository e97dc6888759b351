# quick: full-size records + reuse parity tests, bench n = 12, 11, 10, launch list at n = 12
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TAG=${1:-quick}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${TAG}_build.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_fullsize.py tests/test_gpu_parity.py -x -q --timeout 300 -k "bench or nofoldfp or reuse or saturating or symmetry" > gpurun_out/${TAG}_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/${TAG}_pytest.log
for n in 12 11 10; do timeout 300 python bench.py --n $n --no-cpu-baseline > gpurun_out/${TAG}_n$n.log 2>&1; done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches.csv python bench.py --n 12 --steps 1 --warmup 0 --no-cpu-baseline > gpurun_out/${TAG}_ncu2.log 2>&1
