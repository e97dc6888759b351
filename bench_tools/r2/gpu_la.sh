# lookahead at n = 12 (forced) vs default; n = 13
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TAG=${1:-la}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${TAG}_build.log 2>&1
timeout 300 python bench.py --n 12 --no-cpu-baseline > gpurun_out/${TAG}_n12.log 2>&1
MP_LOOKAHEAD=2 timeout 300 python bench.py --n 12 --no-cpu-baseline > gpurun_out/${TAG}_n12_la.log 2>&1
timeout 600 python bench.py --n 13 --no-cpu-baseline --steps 3 --warmup 1 > gpurun_out/${TAG}_n13.log 2>&1
MP_LOOKAHEAD=2 timeout 600 python bench.py --n 13 --no-cpu-baseline --steps 3 --warmup 1 > gpurun_out/${TAG}_n13_la.log 2>&1
