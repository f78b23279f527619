#!/bin/bash
for v in main fwp8 fwp2; do
  lib=""; [ "$v" != "main" ] && lib="TVLP_LIB=variants/$v/libtvlp_b200.so"
  echo "=== $v" >> gpurun_out/r2_ab_fwp.log
  env $lib timeout 300 python -m pytest tests -q -m gpu -k "framewise" --timeout 300 2>&1 | grep -E "passed|failed" >> gpurun_out/r2_ab_fwp.log
  env $lib timeout 200 python bench.py --config framewise_b32_t48000 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('ms', d['ms_per_step'], 'parity', d.get('parity_max_err'), {k: v['us_per_step'] for k, v in d['kernels'].items()})" >> gpurun_out/r2_ab_fwp.log 2>&1
done
