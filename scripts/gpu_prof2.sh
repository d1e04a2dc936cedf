#!/bin/bash
mkdir -p gpurun_out
TAG=${TAG:-r01d}
LSW_TC_STORE=tma timeout 900 ncu --set full --clock-control none --import-source on -k regex:switch_tc -s 1 -c 1 \
  -o gpurun_out/switch_${TAG} python scripts/prof_kernels.py --layers 4 --tokens 3 > gpurun_out/ncu_switch_${TAG}.log 2>&1
tail -3 gpurun_out/ncu_switch_${TAG}.log
