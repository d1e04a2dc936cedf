#!/bin/bash
for cfg in sweep-n8-r16-k3 sweep-n8-r16-k4 sweep-n8-r32-k3 sweep-n8-r64-k2 sweep-n8-r16-k1; do
python scripts/tune_switch.py --config $cfg --layers 8 "order=sweep" "mma2=1" 2>&1 | grep setting | sed "s/^/$cfg /"
done
LSW_TC_MMA2=1 LSW_TC_KERNEL=tg timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_restore.py -q -x -k "tg or r4k4 or r64k3 or restore" 2>&1 | tail -2
