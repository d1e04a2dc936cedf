#!/bin/bash
set -x
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "trajectory" 2>&1 | tail -3
timeout 1200 python scripts/tune_switch.py --repeat 2 "store=tma" "store=stg" "store=tma,astages=3" "store=tma,astages=4" "store=tma,astages=1" 2>&1 | tee gpurun_out/tune8.txt
timeout 300 python scripts/tune_gemv.py 2>&1 | tail -1
