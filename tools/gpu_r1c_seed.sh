#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"
timeout -s KILL 900 python -m pytest tests/test_gpu_lasp2.py tests/test_gpu_peer_exchange.py tests/test_gpu_kernels.py tests/test_gpu_lasp1.py tests/test_gpu_hybrid.py tests/test_gpu_fullsize.py -q -x -p no:cacheprovider 2>&1 | tail -4
timeout -s KILL 300 python tools/cfg5_sweep.py 65536 524288 2097152 2>&1 | grep -A1 "sequential t=7" | grep graph
timeout -s KILL 300 python bench.py --workload cfg3 --no-cpu-baseline --no-secondary 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('cfg3', d['ms_per_step'], d['per_kernel_ms_per_step'])"
LASP2_DEFINES=LASP2_SPAN python -m paper_2502_07563_b200.build > /dev/null 2>&1
for n in 8192 524288; do timeout -s KILL 200 python tools/cta_phase_probe.py $n; done 2>&1
