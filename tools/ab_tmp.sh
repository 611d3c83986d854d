cd "${GRAFT_REPO_ROOT:-.}"
cp ab_so/mask.so paper_2502_07563_b200/liblasp2_b200.so
timeout -s KILL 600 python -m pytest tests/test_gpu_softmax_kernels.py tests/test_gpu_cp.py -m gpu -q -x -p no:cacheprovider 2>&1 | tail -2
for v in base mask base mask base mask; do
cp ab_so/$v.so paper_2502_07563_b200/liblasp2_b200.so
timeout -s KILL 300 python tools/perf_probe.py 0 softmax 32768 2>&1 | tail -1 | sed "s/^/$v /"
done
