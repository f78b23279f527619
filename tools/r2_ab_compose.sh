#!/bin/bash
out=gpurun_out/r2_ab_compose.log; : > $out
timeout 900 python -m pytest tests -q -m gpu -k "config4 or hier or long or 4p8 or 1p44 or split or segment" --timeout 600 2>&1 | tail -2 >> $out
for v in 1 0; do
  echo "=== TVLP_COMPOSE_TREE=$v" >> $out
  TVLP_COMPOSE_TREE=$v timeout 300 python bench.py --config tv_b1_t14400000 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('ms', d['ms_per_step'], 'parity', d.get('parity_max_err'), 'refined', d.get('refined_sequences'), {k: v['us_per_step'] for k, v in d['kernels'].items()})" >> $out 2>&1
done
