# A/B of library builds under build/ab/<variant> (argv: variants), c3 and c4, 3 rounds
for rep in 1 2 3; do for v in "$@"; do for c in c3 c4; do
  echo -n "$v rep$rep "; CSPQ_LIB_PATH=build/ab/$v/libcspq_b200.so timeout 120 python scripts/probe_tc_bits.py $c 0 2>&1 | tail -1
done; done; done
