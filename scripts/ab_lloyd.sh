# A/B of library builds under build/ab/<variant> on the Lloyd training (argv: configs variants...)
cfgs=$1; shift
for rep in 1 2; do for v in "$@"; do
  echo -n "$v rep$rep "; CSPQ_LIB_PATH=build/ab/$v/libcspq_b200.so timeout 300 python scripts/probe_lloyd.py $cfgs 2>&1 | tr '\n' ' ' | sed 's/(assign[^)]*)//g'; echo
done; done
