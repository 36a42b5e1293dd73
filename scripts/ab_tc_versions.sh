timeout 600 python -m pytest tests/test_encode_tc_gpu.py tests/test_encode_gpu.py -x -q 2>&1 | tail -4
for c in c3 c4 c5 c1; do
 for v in 1 2 1 2; do echo -n "v$v "; CSPQ_TC_KERNEL=$v timeout 120 python scripts/probe_tc_bits.py $c 0 2>&1 | tail -1; done
done
