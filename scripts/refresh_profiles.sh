#!/bin/bash
# Re-measure every bench line and the ncu evidence (run on the GPU box via gpurun).
# Outputs land in gpurun_out/ (copied into profiles/ by hand after review).
set -u
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
tag=${1:-r1}
for c in c3 c1 c2 c4 c5; do
  timeout 900 python bench.py --config $c > gpurun_out/${tag}_bench_$c.jsonl 2> gpurun_out/${tag}_bench_$c.err
  echo "bench $c rc=$?" >> gpurun_out/${tag}_status.txt
done
timeout 900 python bench.py --impl reference > gpurun_out/${tag}_bench_c3_reference_arm.jsonl 2> gpurun_out/${tag}_bench_ref.err
echo "ref rc=$?" >> gpurun_out/${tag}_status.txt
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/${tag}_launches.csv \
  python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/${tag}_ncu_launch.log 2>&1
echo "ncu launches rc=$?" >> gpurun_out/${tag}_status.txt
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:encode_tc_kernel --launch-skip 13 -c 1 \
  -o gpurun_out/${tag}_tc_full python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/${tag}_ncu_full.log 2>&1
echo "ncu full rc=$?" >> gpurun_out/${tag}_status.txt
