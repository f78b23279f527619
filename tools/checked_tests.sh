#!/bin/bash
# The GPU test suite against the checked build (device-side bounds/protocol
# assertions, -D TVLP_CHECKED=1): the stand-in for compute-sanitizer where the
# pool has it disabled.  Build first (here or on the box):
#   python -m paper_2406_05128_b200.build --define TVLP_CHECKED=1 --out variants/checked/libtvlp_b200.so
mkdir -p gpurun_out
TVLP_LIB=variants/checked/libtvlp_b200.so timeout 2400 python -m pytest tests -q -m gpu --timeout 900 \
  -p no:cacheprovider > gpurun_out/r2_checked_tests.log 2>&1
echo "exit $?" >> gpurun_out/r2_checked_tests.log
grep -c "TVLP_ASSERT" gpurun_out/r2_checked_tests.log >> gpurun_out/r2_checked_tests.log
for c in tv_b64_t48000 framewise_b32_t48000 hpn_b32_t48000 tv_b1_t14400000; do
  TVLP_LIB=variants/checked/libtvlp_b200.so timeout 600 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 | cut -c1-200 >> gpurun_out/r2_checked_tests.log
done
