#!/bin/bash
TRACE_ARGS="--B 8" BENCH_ARGS="--shard-of 8" bash tools/chain_ab.sh r2_ab_st_b8 main st4 st6
bash tools/chain_ab.sh r2_ab_st_b64 main st4 st6
