# A/B: every library under variants/*/ against the in-tree build on all bench
# configs (ms_per_step; e2e and the CPU baseline skipped where possible)
for cfg in ${CFGS:-tv_b64_t48000 tv_b4_t24000 framewise_b32_t48000 tv_b1_t14400000 tv_frames_b64_t48000 hpn_b32_t48000}; do
  for d in main variants/*/; do
    n=$(basename $d)
    if [ "$n" = main ]; then lib=""; else lib="$d/libtvlp_b200.so"; fi
    TVLP_LIB=$lib timeout 300 python bench.py --config $cfg --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/ab_${cfg}_$n.log 2>&1
    echo -n "$cfg $n "; tail -n 1 gpurun_out/ab_${cfg}_$n.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d.get('e2e',{}).get('ms_per_step'))"
  done
done
