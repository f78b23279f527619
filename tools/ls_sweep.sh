for cfg in tv_b64_t48000 tv_b4_t24000; do for ls in 160 240 320 384 480 640 960; do
echo -n "$cfg Ls=$ls "; TVLP_SUBCHUNK=$ls timeout 300 python bench.py --config $cfg --steps 10 --warmup 3 --no-cpu-baseline 2>&1 | tail -n 1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], {k:v['us_per_step'] for k,v in d['kernels'].items() if k in ('basis','carry_fwd','apply_fwd','adjoint_zs','carry_bwd','adjoint_apply')})"
done; done
