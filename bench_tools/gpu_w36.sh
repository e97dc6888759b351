cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "large_n" > gpurun_out/w36_large.log 2>&1; echo "rc=$?" >> gpurun_out/w36_large.log
