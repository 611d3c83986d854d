cd "${GRAFT_REPO_ROOT:-.}"
for v in base nohint base nohint; do
cp ab_so/$v.so paper_2502_07563_b200/liblasp2_b200.so
timeout -s KILL 300 python tools/perf_probe.py 0 softmax 32768 2>&1 | tail -1 | sed "s/^/$v /"
timeout -s KILL 300 python tools/masked_bwd_probe.py 524288 2>&1 | head -1 | sed "s/^/$v /"
timeout -s KILL 300 python tools/rank_probe.py 16384 8 0 2>&1 | tail -1 | sed "s/^/$v /"
done
