#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout -s KILL 600 python -m pytest tests/test_gpu_softmax_kernels.py tests/test_gpu_cp.py -q -x -p no:cacheprovider > gpurun_out/t_poly.log 2>&1; echo "rc=$?" >> gpurun_out/t_poly.log
tail -3 gpurun_out/t_poly.log
for pf in 16 12 10 8; do
  LASP2_DEFINES="LASP2_POLY_FROM=$pf" python -m paper_2502_07563_b200.build > /dev/null 2>&1
  echo "POLY_FROM=$pf"; timeout -s KILL 300 python tools/perf_probe.py 0 softmax 32768 2>&1 | grep fwd
done
