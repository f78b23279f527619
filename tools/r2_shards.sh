#!/bin/bash
# per-GPU shares of config 3's strong split, measured on one GPU
mkdir -p gpurun_out
for s in 8 4 2; do
  timeout 300 python bench.py --steps 50 --warmup 5 --shard-of $s --no-cpu-baseline > gpurun_out/r2_shard$s.json 2> gpurun_out/r2_shard$s.err
done
timeout 300 python bench.py --steps 50 --warmup 5 --config tv_b4_t24000 --no-cpu-baseline > gpurun_out/r2_cfg1.json 2> gpurun_out/r2_cfg1.err
