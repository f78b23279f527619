# A/B the tuning variants under variants/*/ on the default bench config
for d in variants/*/; do
  n=$(basename $d)
  TVLP_LIB=$d/libtvlp_b200.so timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/v_$n.log 2>&1
  echo -n "$n "; tail -1 gpurun_out/v_$n.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], {k:v['us_per_step'] for k,v in d['kernels'].items() if k in ('basis','apply_fwd','adjoint_apply')})"
done
echo -n "main "; timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], {k:v['us_per_step'] for k,v in d['kernels'].items() if k in ('basis','apply_fwd','adjoint_apply')})"
