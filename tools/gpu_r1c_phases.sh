#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout -s KILL 900 python -m pytest tests/test_gpu_lasp2.py tests/test_gpu_peer_exchange.py tests/test_gpu_acceptance.py tests/test_gpu_clock.py tests/test_gpu_harness.py tests/test_gpu_kernels.py -q -x -p no:cacheprovider 2>&1 | tail -15
timeout -s KILL 300 python tools/cfg5_sweep.py --unmasked 131072 1048576 2>&1 | grep -A1 "t=7"
