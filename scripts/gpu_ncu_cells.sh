#!/bin/bash
# ncu --set full of one switch pass for representative sweep cells and the 13B shape (2-layer slices)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_nc.log 2>&1 || tail -20 gpurun_out/build_nc.log
for rk in "16 2" "16 4" "32 3" "64 2" "64 4"; do set -- $rk
  timeout 600 ncu --set full --clock-control none -k regex:switch_ -s 1 -c 1 -o gpurun_out/cell_r$1k$2 \
    python scripts/prof_kernels.py --layers 2 --tokens 3 --rank $1 --topk $2 > gpurun_out/ncu_cell_r$1k$2.log 2>&1
done
timeout 600 ncu --set full --clock-control none -k regex:switch_ -s 1 -c 1 -o gpurun_out/cell_13b \
    python scripts/prof_kernels.py --config llama2-13b --layers 2 --tokens 3 > gpurun_out/ncu_cell_13b.log 2>&1
ls gpurun_out/*.ncu-rep
