#!/bin/bash
# every bench config once (no CPU leg): gpurun_out/${1}_<config>.json
p=${1:-r2_all}
for c in tv_b64_t48000 tv_b4_t24000 framewise_b32_t48000 tv_b1_t14400000 hpn_b32_t48000 tv_frames_b64_t48000; do
  timeout 300 python bench.py --config $c --no-cpu-baseline > gpurun_out/${p}_$c.json 2> gpurun_out/${p}_$c.err
done
timeout 300 python bench.py --shard-of 8 --no-cpu-baseline > gpurun_out/${p}_shard8.json 2> gpurun_out/${p}_shard8.err
