# tiles per row group (CSPQ_TC_GS debug override) on the in-tree library; argv: "gs list" "config list"
cd "${GRAFT_REPO_ROOT:-/root/repo}"
for rep in 1 2 3; do for g in ${1:-4 6 8 12}; do for c in ${2:-c3 c5 c2}; do
  echo -n "gs$g rep$rep "; CSPQ_TC_GS=$g python scripts/probe_tc_bits.py $c 0 2>&1 | tail -1
done; done; done
