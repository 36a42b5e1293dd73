cd "${GRAFT_REPO_ROOT:-/root/repo}"
for rep in 1 2 3; do for g in 8 16 32; do for c in c3 c4 c5 c1; do
  echo -n "gs$g rep$rep "; CSPQ_TC_GS=$g CSPQ_LIB_PATH=build/ab/gs/libcspq_b200.so python scripts/probe_tc_bits.py $c 0 2>&1 | tail -1
done; done; done
