cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 1 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/w33_torchrun1.log 2>&1; echo "rc=$?" >> gpurun_out/w33_torchrun1.log
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29534 bench.py --impl reference --gpus 1 --steps 2 --warmup 3 > gpurun_out/w33_torchrun1_ref.log 2>&1; echo "rc=$?" >> gpurun_out/w33_torchrun1_ref.log
