#!/bin/bash
bash tools/chain_ab.sh r2_ab_st2_b64 main st2 fst2
TRACE_ARGS="--B 8" BENCH_ARGS="--shard-of 8" bash tools/chain_ab.sh r2_ab_st2_b8 main st2
