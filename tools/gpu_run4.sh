#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout -s KILL 600 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_lasp2.py tests/test_gpu_graph.py -q -x -p no:cacheprovider > gpurun_out/t4.log 2>&1
timeout -s KILL 300 python tools/perf_probe.py 524288 > gpurun_out/perf4.log 2>&1
timeout -s KILL 300 python tools/perf_probe.py 0 softmax 32768 > gpurun_out/perf4_softmax.log 2>&1
timeout -s KILL 600 python bench.py --steps 20 --warmup 5 > gpurun_out/bench4.json 2> gpurun_out/bench4.err
B="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-secondary --eager"
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:tc_apply -s 4 -c 1 -o gpurun_out/b4_cfg2_apply $B --workload cfg2 > gpurun_out/b4_ncu1.log 2>&1
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:tc_causal -s 4 -c 1 -o gpurun_out/b4_cfg3_causal $B --workload cfg3 > gpurun_out/b4_ncu2.log 2>&1
timeout -s KILL 600 ncu --set full --clock-control none -k regex:tc_segment -s 4 -c 1 -o gpurun_out/b4_cfg3_segment $B --workload cfg3 > gpurun_out/b4_ncu3.log 2>&1
timeout -s KILL 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/b4_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
tail -3 gpurun_out/t4.log
