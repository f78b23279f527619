for d in variants/*/ main; do
  n=$(basename $d)
  if [ "$n" = main ]; then lib=""; else lib="$d/libtvlp_b200.so"; fi
  echo -n "$n "; TVLP_LIB=$lib timeout 300 python bench.py --config framewise_b32_t48000 --steps 10 --warmup 3 --no-cpu-baseline 2>&1 | tail -n 1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], {k:v['us_per_step'] for k,v in d['kernels'].items()})"
done
