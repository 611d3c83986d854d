cd "${GRAFT_REPO_ROOT:-.}"
for v in base NOOINTER NOPV NOSTORE base; do
cp ab_so/$v.so paper_2502_07563_b200/liblasp2_b200.so
timeout -s KILL 300 python tools/masked_bwd_probe.py 524288 2>&1 | head -1 | sed "s/^/$v /"
done
