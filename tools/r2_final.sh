#!/bin/bash
# End-of-round measurement set (outputs in gpurun_out/, summarised into profiles/)
mkdir -p gpurun_out
p=${1:-r2_final}
for c in tv_b64_t48000 tv_b4_t24000 framewise_b32_t48000 tv_b1_t14400000 hpn_b32_t48000 hpn_full_b32_t48000 tv_frames_b64_t48000; do
  timeout 900 python bench.py --config $c > gpurun_out/${p}_$c.json 2> gpurun_out/${p}_$c.err
done
for s in 2 4 8; do
  timeout 300 python bench.py --shard-of $s --no-cpu-baseline > gpurun_out/${p}_shard$s.json 2> gpurun_out/${p}_shard$s.err
done
timeout 600 python bench.py --impl reference --steps 5 > gpurun_out/${p}_reference.json 2> gpurun_out/${p}_reference.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"^k_" -c 400 --csv \
  --log-file gpurun_out/${p}_launches_tv_b64_t48000.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/${p}_launches.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:"k_basis4|k_fwd_chain|k_bwd_chain" -c 3 \
  -o gpurun_out/${p}_full_tv_b64 python tools/one_step.py tv_b64_t48000 > gpurun_out/${p}_full.log 2>&1
bash tools/r2_profiles.sh
timeout 900 python tools/integration_e2e.py > gpurun_out/${p}_integration_e2e.jsonl 2> gpurun_out/${p}_integration_e2e.err
timeout 600 python tools/decoder_bench.py 32 > gpurun_out/${p}_decoder_bench.jsonl 2> gpurun_out/${p}_decoder_bench.err
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__throughput.avg.pct_of_peak_sustained_elapsed,sm__warps_active.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active \
  --clock-control none -k regex:"k_osc|k_fir|k_mss|k_stft|k_noise|k_frame_ola|k_step|k_spec|k_source" -c 60 --csv --log-file gpurun_out/${p}_ncu_decoder_kernels.csv \
  python tools/decoder_prof.py 32 hpn > gpurun_out/${p}_ncu_decoder.log 2>&1
