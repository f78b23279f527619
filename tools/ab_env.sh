# A/B an environment knob on the bench configs: ENVS="TVLP_X=0 TVLP_X=1" CFGS="..."
for cfg in ${CFGS:-tv_b64_t48000 tv_b4_t24000 tv_frames_b64_t48000 hpn_b32_t48000}; do
  for rep in 1 2; do
  for ev in ${ENVS}; do
    env $ev timeout 300 python bench.py --config $cfg --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/abe_${cfg}_${ev}.log 2>&1
    echo -n "$cfg $ev "; tail -n 1 gpurun_out/abe_${cfg}_${ev}.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d.get('refined_sequences'))"
  done
  done
done
