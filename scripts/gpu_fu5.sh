#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_fu5.log 2>&1 || tail -20 gpurun_out/build_fu5.log
for f in 0 4 8 12; do LSW_FC_FUSED_PROBE=$f timeout 600 python scripts/time_fused.py 2>&1 | tail -1; done
