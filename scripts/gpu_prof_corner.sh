#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_pc.log 2>&1 || tail -20 gpurun_out/build_pc.log
timeout 900 ncu --set full --clock-control none -k regex:switch_ -s 1 -c 1 \
  -o gpurun_out/switch_corner_r64k2 python scripts/prof_kernels.py --layers 2 --tokens 3 --rank 64 --topk 2 > gpurun_out/ncu_corner1.log 2>&1
timeout 900 ncu --set full --clock-control none -k regex:switch_ -s 1 -c 1 \
  -o gpurun_out/switch_corner_r16k2 python scripts/prof_kernels.py --layers 2 --tokens 3 --rank 16 --topk 2 > gpurun_out/ncu_corner2.log 2>&1
tail -3 gpurun_out/ncu_corner1.log
