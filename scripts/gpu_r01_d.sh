#!/bin/bash
# term-group switch: parity + sweep; token GEMV diagnostics
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -x 2>&1 | tail -4
timeout 900 python scripts/sweep_bench.py --ranks 16,32,64 --experts 8 --topk 1,2,3,4 --out gpurun_out/sweep_d.json 2>&1 | grep -o '"cell[^,]*,.*"switch_frac_of_roofline": [0-9.]*\|"cell[^,]*, "error.*'
for tg in 1 2 3; do LSW_TC_TG=$tg timeout 600 python scripts/sweep_bench.py --ranks 16,64 --experts 8 --topk 3 --out gpurun_out/sweep_d_tg$tg.json 2>&1 | grep -o '"cell[^,]*,.*"switch_frac_of_roofline": [0-9.]*\|"cell[^,]*, "error.*' | sed "s/^/tg=$tg /"; done
export LSW_GEMV_TOKEN=1
for f in 0 1; do LSW_GEMV_TOKEN_FLAGS=$f timeout 300 python scripts/tune_gemv.py; done 2>&1 | tee gpurun_out/tune_gemv_d.jsonl
LSW_GEMV_SLOT_KB=64 timeout 300 python scripts/tune_gemv.py 2>&1 | tee -a gpurun_out/tune_gemv_d.jsonl
unset LSW_GEMV_TOKEN
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 | tee gpurun_out/bench_r01j.json
timeout 600 python bench.py --steps 5 --warmup 3 --config llama2-13b --no-cpu-baseline 2>&1 | tail -1 | tee gpurun_out/bench_r01j_13b.json
