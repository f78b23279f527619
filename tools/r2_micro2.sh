#!/bin/bash
cd tools/micro && nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 carry_hop.cu -o carry_hop && ./carry_hop > ../../gpurun_out/r2_micro_hop.log 2>&1
