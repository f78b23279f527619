#!/bin/bash
out=gpurun_out/r2_ab_fuse.log; : > $out
timeout 600 python -m pytest tests -q -m gpu -k "fused or config3 or grouped" --timeout 600 2>&1 | tail -1 >> $out
for v in 0 1; do
  for c in tv_b64_t48000 hpn_b32_t48000; do
    TVLP_FUSE_GRAD_A=$v timeout 200 python bench.py --config $c --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('fuse=$v $c', d['ms_per_step'], d.get('parity_max_err'), {k: v['us_per_step'] for k, v in d['kernels'].items()})" >> $out 2>&1
  done
done
TVLP_FUSE_GRAD_A=1 timeout 300 python tools/chain_trace.py >> $out 2>&1
