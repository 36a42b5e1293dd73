# compute-sanitizer over the hot kernels (scripts/sanitize_slices.py); summaries -> gpurun_out/r2_sanitize_*.log
CS=/usr/local/cuda/bin/compute-sanitizer
for cfg in c3 c4; do
  for tool in memcheck racecheck synccheck initcheck; do
    for which in tensor simt lloyd kpp; do
      timeout 900 $CS --tool $tool --print-limit 20 --error-exitcode 9 python scripts/sanitize_slices.py $cfg $which > gpurun_out/r2_sanitize_${cfg}_${tool}_${which}.log 2>&1
      echo "$cfg $tool $which rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|error' gpurun_out/r2_sanitize_${cfg}_${tool}_${which}.log | tail -2 | tr '\n' ' ')"
    done
  done
done
