#!/bin/bash
mkdir -p gpurun_out
LSW_GEMV_SMEM_KB=110 timeout 300 python scripts/tune_gemv.py 2>&1 | tail -1
LSW_GEMV_SMEM_KB=72 timeout 300 python scripts/tune_gemv.py 2>&1 | tail -1
LSW_GEMV_SMEM_KB=220 timeout 300 python scripts/tune_gemv.py 2>&1 | tail -1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -x -q 2>&1 | tail -2
timeout 900 python bench.py --steps 20 --warmup 5 --no-cpu-baseline 2>&1 | tail -1 | tee gpurun_out/bench_r01g.json
