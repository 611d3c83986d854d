#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout -s KILL 300 python -m pytest tests/test_gpu_kernels.py -q -p no:cacheprovider -x -k "backward_chunk or dkdv or causal" > gpurun_out/t10_k.log 2>&1
timeout -s KILL 900 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/t10_all.log 2>&1
timeout -s KILL 600 python bench.py --steps 20 --warmup 5 > gpurun_out/bench10.json 2> gpurun_out/bench10.err
tail -3 gpurun_out/t10_*.log
