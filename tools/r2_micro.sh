#!/bin/bash
cd tools/micro && nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 apply_lane.cu -o apply_lane && ./apply_lane > ../../gpurun_out/r2_micro_apply.log 2>&1
