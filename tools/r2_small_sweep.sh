#!/bin/bash
# small-batch (strong-split share) plan sweep: B=8 and B=16 at T=48000
mkdir -p gpurun_out; out=gpurun_out/r2_small_sweep.log; : > $out
run() {  # label, env..., shard
  local label=$1; shift; local sh=$1; shift
  env "$@" timeout 120 python bench.py --steps 30 --warmup 5 --shard-of $sh --no-cpu-baseline > gpurun_out/tmp.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/tmp.json'))
print('$label', 'B=%d'%d['config']['B_per_gpu'], d['ms_per_step'], 'par=%.1e'%d['parity_max_err'], {k:v['us_per_step'] for k,v in d['kernels'].items()})" >> $out 2>&1 || echo "$label FAILED" >> $out
}
for sh in 8 4; do
  for ls in 320 240 160 96; do run "chain_ls$ls" $sh TVLP_SUBCHUNK=$ls; done
  for ls in 320 160 96; do
    run "nochain_ls$ls" $sh TVLP_CHAIN=0 TVLP_SUBCHUNK=$ls
    for sm in 16 64; do for gr in 8 32; do
      run "nochain_ls${ls}_sm${sm}_g$gr" $sh TVLP_CHAIN=0 TVLP_SUBCHUNK=$ls TVLP_CARRY_SERIAL_MAX=$sm TVLP_CARRY_GROUP=$gr
    done; done
  done
done
