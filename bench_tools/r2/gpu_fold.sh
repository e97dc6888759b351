# The parents' fold inside k_spmm (level layout, parents staged as entries) vs separate k_fold passes
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TAG=${1:-fold}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${TAG}_build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_fullsize.py -x -q --timeout 300 -k "bench or noreuse" > gpurun_out/${TAG}_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/${TAG}_pytest.log
for n in 12 11 10 9; do
  timeout 300 python bench.py --n $n --no-cpu-baseline --steps 6 > gpurun_out/${TAG}_n$n.log 2>&1
  MP_FOLD_SPMM=0 timeout 300 python bench.py --n $n --no-cpu-baseline --steps 6 > gpurun_out/${TAG}_n${n}_sep.log 2>&1
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches.csv python bench.py --n 12 --steps 1 --warmup 0 --no-cpu-baseline > gpurun_out/${TAG}_ncu2.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_spmm -s 200 -c 3 -o gpurun_out/${TAG}_kspmm -f python bench.py --n 12 --steps 1 --warmup 0 --no-cpu-baseline > gpurun_out/${TAG}_ncu.log 2>&1
