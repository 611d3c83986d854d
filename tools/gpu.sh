#!/bin/bash
# One parametrised runner for the B200 box (replaces the per-session launch scripts).
#
#   gpurun --timeout S -- 'bash tools/gpu.sh STEP [STEP ...]'
#
# Every step writes under gpurun_out/ and is bounded by its own `timeout`, so a
# hung kernel never outlives the call. Steps:
#   bench            python bench.py (N=1 headline line)             -> bench.json
#   bench:ARGS       python bench.py ARGS (commas -> spaces)         -> bench_<n>.json
#   ref              python bench.py --impl reference                -> bench_ref.json
#   launches         ncu launch list of a short bench run            -> launches.csv
#   ncu:REGEX:WL     ncu --set full of kernels matching REGEX in workload WL -> ncu_<WL>.ncu-rep
#   tests            pytest -m gpu (whole suite)                     -> t_gpu_all.log
#   tests:EXPR       pytest -m gpu -k EXPR                           -> t_gpu_k.log
#   smoke            __graft_entry__.py smoke                        -> smoke.log
#   multirank        torchrun 2 ranks over gloo on one GPU (bench)   -> multirank.log
#   tool:SCRIPT,ARGS python tools/SCRIPT ARGS                        -> tool_<SCRIPT>.log
#   ab:WL            A/B of ab_so/old.so vs ab_so/new.so on workload WL
cd "${GRAFT_REPO_ROOT:-.}" || exit 1
mkdir -p gpurun_out
nb=0
for step in "$@"; do
  case "$step" in
    bench)
      timeout -s KILL 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
      tail -c 400 gpurun_out/bench.json; tail -3 gpurun_out/bench.err ;;
    bench:*)
      nb=$((nb + 1)); a="${step#bench:}"; a="${a//,/ }"
      timeout -s KILL 900 python bench.py $a > gpurun_out/bench_$nb.json 2> gpurun_out/bench_$nb.err
      echo "bench_$nb: $a"; tail -c 400 gpurun_out/bench_$nb.json; tail -3 gpurun_out/bench_$nb.err ;;
    ref)
      timeout -s KILL 900 python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
      tail -c 400 gpurun_out/bench_ref.json ;;
    launches)
      timeout -s KILL 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
        --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline \
        > gpurun_out/launches_stdout.json 2> gpurun_out/launches.err
      python tools/launch_summary.py gpurun_out/launches.csv 2>&1 | tail -20 ;;
    ncu:*)
      rest="${step#ncu:}"; re="${rest%%:*}"; wl="${rest#*:}"
      timeout -s KILL 1200 ncu --set full --clock-control none --import-source on -k "regex:$re" -c 4 \
        -o "gpurun_out/ncu_$wl" -f python bench.py --workload "$wl" --steps 1 --warmup 3 --no-cpu-baseline \
        --no-secondary > "gpurun_out/ncu_$wl.log" 2>&1
      tail -3 "gpurun_out/ncu_$wl.log" ;;
    tests)
      timeout -s KILL 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/t_gpu_all.log 2>&1
      echo "pytest rc=$?" >> gpurun_out/t_gpu_all.log; tail -15 gpurun_out/t_gpu_all.log ;;
    tests:*)
      timeout -s KILL 2400 python -m pytest tests -m gpu -q -p no:cacheprovider -k "${step#tests:}" \
        > gpurun_out/t_gpu_k.log 2>&1
      echo "pytest rc=$?" >> gpurun_out/t_gpu_k.log; tail -25 gpurun_out/t_gpu_k.log ;;
    smoke)
      timeout -s KILL 300 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1
      echo "smoke rc=$?" >> gpurun_out/smoke.log; tail -2 gpurun_out/smoke.log ;;
    multirank)
      timeout -s KILL 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
        --master-port 29533 bench.py --gpus 2 --steps 2 --warmup 3 --dist-backend gloo --no-cpu-baseline \
        > gpurun_out/multirank.log 2>&1
      echo "rc=$?" >> gpurun_out/multirank.log; tail -c 1500 gpurun_out/multirank.log ;;
    tool:*)
      a="${step#tool:}"; script="${a%%,*}"; args=""; [[ "$a" == *,* ]] && args="${a#*,}"; args="${args//,/ }"
      timeout -s KILL 1200 python "tools/$script" $args > "gpurun_out/tool_${script%.py}.log" 2>&1
      echo "rc=$?" >> "gpurun_out/tool_${script%.py}.log"; tail -30 "gpurun_out/tool_${script%.py}.log" ;;
    ab:*)
      wl="${step#ab:}"
      for rep in 1 2; do
        for v in old new; do
          cp "ab_so/$v.so" paper_2502_07563_b200/liblasp2_b200.so
          timeout -s KILL 300 python bench.py --workload "$wl" --no-cpu-baseline --no-secondary 2>/dev/null |
            python -c "
import json, sys
d = json.loads(sys.stdin.read().strip().splitlines()[-1])
print('$v', '$wl', round(d['ms_per_step'], 4), {k: round(x, 4) for k, x in d['per_kernel_ms_per_step'].items()},
      d['clocks']['sm_mhz'])"
        done
      done ;;
    *) echo "unknown step $step"; exit 2 ;;
  esac
done
