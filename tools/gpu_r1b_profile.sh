#!/bin/bash
# round-1 (session b) evidence: bench line, reference arm, launch list, ncu --set full of the bench kernels
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout -s KILL 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout -s KILL 400 python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
timeout -s KILL 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv \
   python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/bench_ncu_stdout.json 2> gpurun_out/launches.err
timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:tc_flat_kernel -c 2 \
   -o gpurun_out/r1b_cfg2_flat -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-secondary > gpurun_out/ncu_flat.log 2>&1
timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:"causal_chunk|segment_states" -c 4 \
   -o gpurun_out/r1b_cfg3 -f python bench.py --workload cfg3 --steps 1 --warmup 3 --no-cpu-baseline --no-secondary > gpurun_out/ncu_cfg3.log 2>&1
timeout -s KILL 300 python tools/pcie_probe.py > gpurun_out/pcie.log 2>&1
ls -la gpurun_out; tail -c 300 gpurun_out/bench.json; cat gpurun_out/pcie.log
