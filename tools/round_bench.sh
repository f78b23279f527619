# Full bench sweep for profiles/: default line (with cpu baseline), the
# reference arm, every config, and the ncu launch list of the default step.
set -x
mkdir -p gpurun_out/rb
timeout 900 python bench.py > gpurun_out/rb/default.log 2>&1
timeout 900 python bench.py --impl reference > gpurun_out/rb/reference.log 2>&1
for c in tv_b4_t24000 framewise_b32_t48000 tv_b1_t14400000 hpn_b32_t48000 tv_frames_b64_t48000 tv_b1_t14400000_split; do
  timeout 600 python bench.py --config $c --no-cpu-baseline > gpurun_out/rb/$c.log 2>&1
done
timeout 600 python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/rb/plain2.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"^k_" -c 40 --csv --log-file gpurun_out/rb/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/rb/ncu_launch.log 2>&1
tail -n 1 gpurun_out/rb/*.log | cut -c1-400
