cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TAG=${1:-sncu}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${TAG}_build.log 2>&1
for n in 3 6; do
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_small_run -s 3 -c 1 -o gpurun_out/${TAG}_small_n$n -f python bench.py --n $n --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/${TAG}_ncu_n$n.log 2>&1
done
