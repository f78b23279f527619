#!/bin/bash
out=gpurun_out/r2_ab_ls.log; : > $out
run() { # label env...
  local label=$1; shift
  env "$@" timeout 200 python bench.py --no-cpu-baseline --steps 20 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$label', 'ms', d['ms_per_step'], 'Ls', d['config']['subchunk'], 'parity', d.get('parity_max_err'), {k: v['us_per_step'] for k, v in d['kernels'].items()})" >> $out 2>&1
}
run main
run ls400 TVLP_SUBCHUNK=400
run ls320 TVLP_SUBCHUNK=320
run ls240 TVLP_SUBCHUNK=240
run u16 TVLP_LIB=variants/u16/libtvlp_b200.so
run u16_ls320 TVLP_LIB=variants/u16/libtvlp_b200.so TVLP_SUBCHUNK=320
run u16_ls600 TVLP_LIB=variants/u16/libtvlp_b200.so TVLP_SUBCHUNK=600
rm -f gpurun_out/r2_ab_fwp.log
for v in main fwp8 fwp8d fwp4d; do
  lib=""; [ "$v" != "main" ] && lib="TVLP_LIB=variants/$v/libtvlp_b200.so"
  echo "=== $v" >> gpurun_out/r2_ab_fwp.log
  env $lib timeout 300 python -m pytest tests -q -m gpu -k "framewise" --timeout 300 2>&1 | grep -E "passed|failed|Error" | head -3 >> gpurun_out/r2_ab_fwp.log
  env $lib timeout 200 python bench.py --config framewise_b32_t48000 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('ms', d['ms_per_step'], 'parity', d.get('parity_max_err'), {k: v['us_per_step'] for k, v in d['kernels'].items()})" >> gpurun_out/r2_ab_fwp.log 2>&1
done
