#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -x -q 2>&1 | tail -2
timeout 600 python scripts/trace_switch.py 2>&1 | grep -B3 -A16 "CTA 49:"
timeout 900 python bench.py --steps 20 --warmup 5 --no-cpu-baseline 2>&1 | tail -1 | tee gpurun_out/bench_r01f.json
timeout 1500 python scripts/tune_switch.py --repeat 2 "order=sweep,chunk=24" "order=sweep,chunk=48" "order=sweep,chunk=64" "order=sweep,chunk=32,store=stg" 2>&1
