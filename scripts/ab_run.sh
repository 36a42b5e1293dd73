#!/bin/bash
# Alternate builds under build/ab/ (AB_VARIANTS, default "a b") on the same box; argv = configs
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
cfgs=${@:-c3 c4}
for rep in 1 2 3; do for v in ${AB_VARIANTS:-a b}; do for c in $cfgs; do
  echo -n "$v rep$rep "; CSPQ_LIB_PATH=build/ab/$v/libcspq_b200.so python scripts/probe_tc_bits.py $c 0 2>&1 | tail -1
done; done; done
