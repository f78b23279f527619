# A/B the tuning variants under variants/*/ on the default bench config
for d in variants/*/ main; do
  n=$(basename $d)
  if [ "$n" = main ]; then lib=""; else lib="$d/libtvlp_b200.so"; fi
  TVLP_LIB=$lib timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/v_$n.log 2>&1
  echo -n "$n "; tail -n 1 gpurun_out/v_$n.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], {k:v['us_per_step'] for k,v in d['kernels'].items() if k in ('basis','carry_fwd','carry_bwd')})"
done
