#!/bin/bash
for rep in 1 2; do
python scripts/tune_switch.py --lib build/bs_4bf23d2/liblsw.so "order=sweep" 2>&1 | grep setting | sed "s/^/prev /"
python scripts/tune_switch.py "order=sweep" 2>&1 | grep setting | sed 's/^/HEAD /'
done
timeout 600 python -m pytest tests/test_gpu_fused.py tests/test_gpu_restore.py -q -x 2>&1 | tail -1
timeout 600 python scripts/time_fused.py
