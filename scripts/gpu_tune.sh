#!/bin/bash
set -x
mkdir -p gpurun_out
TAG=${TAG:-r01b}
LSW_GEMV=ldg timeout 300 python scripts/tune_gemv.py 2>&1 | tail -2
LSW_GEMV=bulk timeout 300 python scripts/tune_gemv.py 2>&1 | tail -2
timeout 900 python scripts/tune_switch.py "order=strip" "order=strip,probe=1" "order=strip,probe=2" 2>&1 | tee gpurun_out/tune3.txt
timeout 900 ncu --set full --clock-control none --import-source on -k regex:switch_tc -s 1 -c 1 \
  -o gpurun_out/switch_${TAG} python scripts/prof_kernels.py --layers 4 --tokens 3 > gpurun_out/ncu_switch_${TAG}.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemv -s 4 -c 4 \
  -o gpurun_out/gemv_${TAG} python scripts/prof_kernels.py --layers 4 --tokens 3 > gpurun_out/ncu_gemv_${TAG}.log 2>&1
