#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
P="python tools/perf_probe.py 524288"
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:tc_causal_chunk_kernel -s 3 -c 1 -o gpurun_out/p6_causal $P > /dev/null 2>&1
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:"tc_causal_chunk_kernel<true>" -s 2 -c 1 -o gpurun_out/p6_pair $P > /dev/null 2>&1
S="python tools/perf_probe.py 0 softmax 16384"
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:tc_softmax_fwd -s 2 -c 1 -o gpurun_out/p6_smfwd $S > /dev/null 2>&1
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:tc_softmax_bwd -s 2 -c 1 -o gpurun_out/p6_smbwd $S > /dev/null 2>&1
ls -la gpurun_out/
