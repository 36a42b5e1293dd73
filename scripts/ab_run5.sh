cd "${GRAFT_REPO_ROOT:-/root/repo}"
for rep in 1 2 3 4 5; do for v in s0 s100 s200; do for c in c3 c5 c2; do
  echo -n "$v rep$rep "; CSPQ_LIB_PATH=build/ab/$v/libcspq_b200.so python scripts/probe_tc_bits.py $c 0 2>&1 | tail -1
done; done; done
