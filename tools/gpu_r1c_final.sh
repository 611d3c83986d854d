#!/bin/bash
# session-c evidence refresh: bench line, reference arm, launch list, ncu --set full of the bench kernels
# and of the LASP-2H kernels, full GPU test suite
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout -s KILL 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout -s KILL 400 python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
timeout -s KILL 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv \
   python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/bench_ncu_stdout.json 2> gpurun_out/launches.err
timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:tc_flat_kernel -c 2 \
   -o gpurun_out/r1c_cfg2_flat -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-secondary > gpurun_out/ncu_flat.log 2>&1
timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:"causal_chunk|segment_states" -c 4 \
   -o gpurun_out/r1c_cfg3 -f python bench.py --workload cfg3 --steps 1 --warmup 3 --no-cpu-baseline --no-secondary > gpurun_out/ncu_cfg3.log 2>&1
timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:"tc_softmax" -c 2 \
   -o gpurun_out/r1c_softmax -f python tools/perf_probe.py 0 softmax 32768 > gpurun_out/ncu_softmax.log 2>&1
timeout -s KILL 300 python tools/perf_probe.py 0 softmax 32768 > gpurun_out/perf_softmax.log 2>&1
timeout -s KILL 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/t_gpu_all.log 2>&1; echo "pytest rc=$?" >> gpurun_out/t_gpu_all.log
timeout -s KILL 300 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
ls -la gpurun_out; tail -c 400 gpurun_out/bench.json; tail -2 gpurun_out/t_gpu_all.log; tail -1 gpurun_out/smoke.log; cat gpurun_out/perf_softmax.log
