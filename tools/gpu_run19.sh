#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout -s KILL 600 python -m pytest tests/test_gpu_kernels.py -q -p no:cacheprovider -x -k "nomask_local" > gpurun_out/t19a.log 2>&1
tail -3 gpurun_out/t19a.log
timeout -s KILL 600 python -m pytest tests/test_gpu_lasp2.py -q -p no:cacheprovider -x > gpurun_out/t19b.log 2>&1
tail -3 gpurun_out/t19b.log
timeout -s KILL 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-secondary > gpurun_out/bench19.json 2> gpurun_out/bench19.err
cat gpurun_out/bench19.json | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print(d['value'], d['ms_per_step'], d.get('per_kernel_ms_per_step'), d['roofline'])"
