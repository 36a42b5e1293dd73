#!/bin/bash
# Alternate two builds (build/ab/a, build/ab/b) on the same box: argv = configs (default c3 c4)
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
cfgs=${@:-c3 c4}
for rep in 1 2 3; do for v in a b; do for c in $cfgs; do
  echo -n "$v rep$rep "; CSPQ_LIB_PATH=build/ab/$v/libcspq_b200.so python scripts/probe_tc_bits.py $c 0 2>&1 | tail -1
done; done; done
