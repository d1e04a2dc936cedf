#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null || exit 1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:switch_fc_kernel -c 4 \
   -o gpurun_out/prof_fused python scripts/prof_fused.py > gpurun_out/prof_fused.log 2>&1; echo "ncu rc=$?"
tail -3 gpurun_out/prof_fused.log
ls -la gpurun_out/prof_fused.ncu-rep
