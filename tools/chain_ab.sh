#!/bin/bash
# A/B of chained-kernel variants on the GPU box: trace + bench step time.
# usage: tools/chain_ab.sh out_prefix [variant[:ENV=V ...]] ...   ("main" = the product library)
out=$1; shift
for spec in "$@"; do
  v=${spec%%:*}; envs=""
  [ "$spec" != "$v" ] && envs=$(echo ${spec#*:} | tr ',' ' ')
  lib=""; [ "$v" != "main" ] && lib="TVLP_LIB=variants/$v/libtvlp_b200.so"
  echo "=== $spec" >> gpurun_out/${out}.log
  env $lib $envs timeout 120 python tools/chain_trace.py $TRACE_ARGS >> gpurun_out/${out}.log 2>&1
  env $lib $envs timeout 200 python bench.py --no-cpu-baseline --steps 10 $BENCH_ARGS 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('ms', d['ms_per_step'], 'parity', d.get('parity_max_err'), {k: v['us_per_step'] for k, v in d['kernels'].items()})" >> gpurun_out/${out}.log 2>&1
done
