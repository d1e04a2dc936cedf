#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "trajectory or many_tiles or gemv" 2>&1 | tail -2
LSW_GEMV_SMEM_KB=220 timeout 300 python scripts/tune_gemv.py 2>&1 | tail -1
LSW_GEMV_SMEM_KB=110 timeout 300 python scripts/tune_gemv.py 2>&1 | tail -1
LSW_GEMV_SMEM_KB=72 timeout 300 python scripts/tune_gemv.py 2>&1 | tail -1
timeout 1500 python scripts/tune_switch.py --repeat 2 "chunk=48" "chunk=48,astages=2" "chunk=32,astages=2" "chunk=96,astages=2" 2>&1
