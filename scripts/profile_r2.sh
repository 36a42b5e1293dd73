#!/bin/bash
# Round-2 evidence (run on the GPU box via gpurun): GPU tests, the default bench line, the ncu
# launch list of the default bench, full ncu captures of the c3 and c4 encode launches and of
# one Lloyd iteration's kernels (c2).  Outputs in gpurun_out/ (summaries copied into profiles/).
set -u
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
tag=${1:-r2}
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/${tag}_gputests.log 2>&1; echo "gpu tests rc=$? $(tail -1 gpurun_out/${tag}_gputests.log)"
timeout 1200 python bench.py > gpurun_out/${tag}_bench.jsonl 2> gpurun_out/${tag}_bench.err; echo "bench rc=$?"
# launch list of the headline bench (no e2e / CPU / extras: the device-resident steps)
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/${tag}_launches_c3.csv \
  python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-extra > gpurun_out/${tag}_ncu_launch.log 2>&1; echo "launch list rc=$?"
# full captures of the encode launches (prof_tc.py: data + sampled codebooks, 2 encodes; capture the second)
timeout 900 ncu --set full --import-source on --clock-control none -k regex:encode_tc_kernel -s 1 -c 1 \
  -o gpurun_out/${tag}_ncu_full_c3 python scripts/prof_tc.py c3 10000000 > gpurun_out/${tag}_ncu_full_c3.log 2>&1; echo "full c3 rc=$?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:encode_tc_kernel -s 1 -c 1 \
  -o gpurun_out/${tag}_ncu_full_c4 python scripts/prof_tc.py c4 50000000 > gpurun_out/${tag}_ncu_full_c4.log 2>&1; echo "full c4 rc=$?"
# Lloyd (c2 training): launch list and a full capture of the settle / sums kernels of one iteration
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${tag}_launches_lloyd_c2.csv \
  python scripts/probe_lloyd.py c2 > gpurun_out/${tag}_ncu_lloyd_launch.log 2>&1; echo "lloyd launch list rc=$?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"tc_settle|sums_kernel|scatter_kernel" -s 30 -c 3 \
  -o gpurun_out/${tag}_ncu_full_lloyd_c2 python scripts/probe_lloyd.py c2 > gpurun_out/${tag}_ncu_full_lloyd.log 2>&1; echo "full lloyd rc=$?"
