cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python __graft_entry__.py smoke > gpurun_out/w34_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/w34_smoke.log
timeout 600 python -m pytest tests/test_gpu_sharded.py -q -x > gpurun_out/w34_sharded.log 2>&1; echo "rc=$?" >> gpurun_out/w34_sharded.log
