#!/bin/bash
# Per-config ncu summaries of one bench step (tools/one_step.py) and the launch
# list of the default bench command; outputs under gpurun_out/ (copied to profiles/).
mkdir -p gpurun_out
MET=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__throughput.avg.pct_of_peak_sustained_elapsed,sm__warps_active.avg.pct_of_peak_sustained_active,launch__grid_size,launch__block_size,launch__registers_per_thread,smsp__inst_executed.sum,sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active
for c in ${@:-tv_b64_t48000 tv_b4_t24000 framewise_b32_t48000 tv_b1_t14400000 hpn_b32_t48000 tv_frames_b64_t48000}; do
  timeout 900 ncu --profile-from-start off --clock-control none --metrics $MET --csv \
    --log-file gpurun_out/r2_ncu_$c.csv python tools/one_step.py $c > gpurun_out/r2_ncu_$c.log 2>&1
done
timeout 600 ncu --profile-from-start off --clock-control none --metrics $MET --csv \
  --log-file gpurun_out/r2_ncu_tv_b64_t48000_shard8.csv python tools/one_step.py tv_b64_t48000 --shard-of 8 > /dev/null 2>&1
