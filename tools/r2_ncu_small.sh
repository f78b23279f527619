#!/bin/bash
# ncu of one fwd+bwd step at config 3's 8-way share (B=8, T=48000)
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"^k_" -s 20 -c 6 \
  -o gpurun_out/r2_small_b8 python bench.py --steps 2 --warmup 3 --shard-of 8 --no-cpu-baseline > gpurun_out/r2_ncu_small.log 2>&1
