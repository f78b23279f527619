#!/bin/bash
out=gpurun_out/r2_ab_prega.log; : > $out
for rep in 1 2; do
for v in main pre_ga; do
  lib=""; [ "$v" != "main" ] && lib="TVLP_LIB=variants/$v/libtvlp_b200.so"
  for a in "" "--shard-of 8"; do
    env $lib timeout 200 python bench.py $a --no-cpu-baseline --steps 30 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v $a', d['ms_per_step'], {k: v['us_per_step'] for k, v in d['kernels'].items()})" >> $out 2>&1
  done
done
done
