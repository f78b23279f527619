#!/bin/bash
out=gpurun_out/r2_ls_small.log; : > $out
for ls in 96 120 160 200 240 320 480; do
  for args in "--config tv_b4_t24000" "--shard-of 8" "--shard-of 4"; do
    TVLP_SUBCHUNK=$ls timeout 200 python bench.py $args --no-cpu-baseline --steps 30 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('ls=$ls', '$args', d['config']['subchunk'], d['ms_per_step'], d.get('parity_max_err'))" >> $out 2>&1
  done
done
