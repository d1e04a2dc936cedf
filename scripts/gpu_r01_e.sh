#!/bin/bash
python scripts/tune_switch.py --repeat 2 "order=sweep" "w4d=1" "probe=1" "probe=1,w4d=1" 2>&1 | grep setting
LSW_TC_W4D=1 LSW_TC_KERNEL=v1 timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "trajectory or many_tiles" 2>&1 | tail -2
