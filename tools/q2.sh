for cfg in "256 32" "16 10" "16 5" "8 4"; do set -- $cfg
echo -n "serial<=$1 group=$2: "; TVLP_CARRY_SERIAL_MAX=$1 TVLP_CARRY_GROUP=$2 timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline 2>&1 | tail -n 1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['refined_sequences'], {k:v['us_per_step'] for k,v in d['kernels'].items() if 'carry' in k or 'refine' in k or 'compose' in k})"
done
