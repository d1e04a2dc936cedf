#!/bin/bash
# Bench + launch list under gpurun (1 GPU).
set -x
mkdir -p gpurun_out
timeout 600 python bench.py --steps 20 --warmup 5 ${BENCH_ARGS} 2>&1 | tail -5 | tee gpurun_out/bench.jsonl
