#!/bin/bash
# whole-token GEMV: tests + timing; switch accumulator modes for > 4 terms
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x 2>&1 | tail -4
for kb in 32 16 48; do LSW_GEMV_SLOT_KB=$kb timeout 300 python scripts/tune_gemv.py; done 2>&1 | tee gpurun_out/tune_gemv_c.jsonl
LSW_GEMV_SMEM_KB=160 timeout 300 python scripts/tune_gemv.py 2>&1 | tee -a gpurun_out/tune_gemv_c.jsonl
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 | tee gpurun_out/bench_r01i.json
for sp in 0 1; do LSW_TC_SPLIT=$sp timeout 900 python scripts/sweep_bench.py --ranks 16,32 --experts 8 --topk 2,3,4 --out gpurun_out/sweep_split$sp.json 2>&1 | tail -6; done
LSW_TC_NSUB=1 timeout 900 python scripts/sweep_bench.py --ranks 16,32 --experts 8 --topk 2,3,4 --out gpurun_out/sweep_nsub1.json 2>&1 | tail -6
