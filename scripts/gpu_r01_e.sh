#!/bin/bash
python scripts/tune_switch.py "order=sweep" 2>&1 | grep setting | sed 's/^/v1 /'
LSW_TC_KERNEL=tg python scripts/tune_switch.py "order=sweep" 2>&1 | grep setting | sed 's/^/tg /'
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -x 2>&1 | tail -3
timeout 900 python scripts/sweep_bench.py --ranks 16,32,64 --experts 8 --topk 1,2,3,4 --out gpurun_out/sweep_g.json 2>&1 | grep -o '"cell[^,]*,.*"switch_frac_of_roofline": [0-9.]*\|"cell[^,]*, "error.*' | cut -c1-30,190-
LSW_TC_KERNEL=tg timeout 900 python scripts/sweep_bench.py --ranks 16,32 --experts 8 --topk 1,2 --out gpurun_out/sweep_g_tg.json 2>&1 | grep -o '"cell[^,]*,.*"switch_frac_of_roofline": [0-9.]*\|"cell[^,]*, "error.*' | cut -c1-30,190- | sed 's/^/tg /'
