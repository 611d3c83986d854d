#!/bin/bash
# N>1 plumbing on one GPU: torchrun 2 ranks over gloo (NCCL refuses two ranks on one device)
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout -s KILL 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 \
  bench.py --gpus 2 --steps 2 --warmup 3 --dist-backend gloo --no-cpu-baseline > gpurun_out/multirank.log 2>&1
echo "rc=$?" >> gpurun_out/multirank.log
tail -c 1500 gpurun_out/multirank.log
timeout -s KILL 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29534 \
  bench.py --gpus 2 --steps 2 --warmup 3 --dist-backend gloo --no-cpu-baseline --impl reference > gpurun_out/multirank_ref.log 2>&1
echo "rc=$?" >> gpurun_out/multirank_ref.log
tail -c 600 gpurun_out/multirank_ref.log
