#!/bin/bash
# compute-sanitizer over every kernel family (tools/sanitize_driver.py);
# logs -> gpurun_out/r2_sanitize_<tool>.log, summary -> gpurun_out/r2_sanitize_summary.txt
# usage (GPU box): bash tools/sanitize.sh [tool ...]
mkdir -p gpurun_out
CS=/usr/local/cuda/bin/compute-sanitizer
FAMS="chain chain_ref grouped ti f64 frames framewise stepup"
tools=${@:-memcheck racecheck synccheck initcheck}
sum=gpurun_out/r2_sanitize_summary.txt; : > $sum
for tool in $tools; do
  log=gpurun_out/r2_sanitize_$tool.log; : > $log
  for fam in $FAMS hier; do
    extra=""
    [ "$fam" = hier ] && extra="TVLP_CARRY_SERIAL_MAX=16 TVLP_CARRY_GROUP=8"
    echo "=== $tool $fam" >> $log
    env $extra PYTORCH_NO_CUDA_MEMORY_CACHING=1 timeout 900 $CS --tool $tool --error-exitcode 9 python tools/sanitize_driver.py $fam >> $log 2>&1
    rc=$?
    echo "$tool $fam rc=$rc $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY' $log | tail -1)" >> $sum
  done
done
cat $sum
