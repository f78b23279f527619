for ls in 480 240; do
echo -n "tvf Ls=$ls "; TVLP_SUBCHUNK=$ls timeout 300 python bench.py --config tv_frames_b64_t48000 --steps 10 --warmup 3 --no-cpu-baseline 2>&1 | tail -n 1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['config']['subchunk'], {k:v['us_per_step'] for k,v in d['kernels'].items() if k in ('basis','carry_fwd','apply_fwd','adjoint_zs','carry_bwd','adjoint_apply','grad_frames','compose')})"
done
