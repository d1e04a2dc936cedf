#!/bin/bash
# ncu captures under gpurun (1 GPU).  Never a multi-rank command.
set -x
mkdir -p gpurun_out
TAG=${TAG:-r01}
# 1) launch list of the bench's timed tokens (cold-cache, serialised: compare shares)
#    create packs 7 kernels; 3 warm-up tokens x (2 + 4*32) launches precede the timed ones.
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -s 397 -c 260 --csv \
  --log-file gpurun_out/launches_${TAG}.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch_${TAG}.log 2>&1
# 2) full set on the switch kernel (second launch = fused switch mode) and one GEMV of each group
timeout 900 ncu --set full --clock-control none --import-source on -k regex:switch_tc -s 1 -c 1 \
  -o gpurun_out/switch_${TAG} python scripts/prof_kernels.py --layers 4 --tokens 3 > gpurun_out/ncu_switch_${TAG}.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemv -s 4 -c 4 \
  -o gpurun_out/gemv_${TAG} python scripts/prof_kernels.py --layers 4 --tokens 3 > gpurun_out/ncu_gemv_${TAG}.log 2>&1
ls -la gpurun_out
