#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout -s KILL 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 \
   bench.py --gpus 2 --steps 3 --warmup 3 --dist-backend gloo > gpurun_out/bench15_n2.json 2> gpurun_out/bench15_n2.err
timeout -s KILL 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29512 \
   bench.py --impl reference --gpus 2 --steps 2 --warmup 3 > gpurun_out/bench15_ref_n2.json 2> gpurun_out/bench15_ref_n2.err
timeout -s KILL 600 python bench.py --workload cfg4 --seq-len 32768 --steps 5 --warmup 3 --no-secondary > gpurun_out/bench15_cfg4.json 2> gpurun_out/bench15_cfg4.err
tail -5 gpurun_out/bench15_n2.err
