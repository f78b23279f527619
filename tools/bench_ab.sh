#!/bin/bash
# A/B of library variants / env knobs on the bench step (no trace).
# usage: tools/bench_ab.sh out_prefix [variant[:ENV=V,...]] ...   ("main" = the product library)
out=$1; shift
for spec in "$@"; do
  v=${spec%%:*}; envs=""
  [ "$spec" != "$v" ] && envs=$(echo ${spec#*:} | tr ',' ' ')
  lib=""; [ "$v" != "main" ] && lib="TVLP_LIB=variants/$v/libtvlp_b200.so"
  for rep in 1 2; do
  env $lib $envs timeout 200 python bench.py --no-cpu-baseline --steps 20 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$spec', 'ms', d['ms_per_step'], 'parity', d.get('parity_max_err'), 'sub', d['config']['subchunk'], {k: v['us_per_step'] for k, v in d['kernels'].items()})" >> gpurun_out/${out}.log 2>&1
  done
done
