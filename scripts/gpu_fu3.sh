#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_fu3.log 2>&1 || tail -20 gpurun_out/build_fu3.log
timeout 600 python scripts/time_fused.py 2>&1 | tail -1
LSW_FC_STAGES=3 LSW_FC_BBUFS=2 LSW_FC_ASTAGES=3 timeout 600 python scripts/time_fused.py 2>&1 | tail -1
LSW_FC_STAGES=3 LSW_FC_BBUFS=2 LSW_FC_ASTAGES=3 LSW_FC_FUSED_PROBE=4 timeout 600 python scripts/time_fused.py 2>&1 | tail -1
LSW_FC_STAGES=4 LSW_FC_BBUFS=2 LSW_FC_ASTAGES=2 timeout 600 python scripts/time_fused.py 2>&1 | tail -1
timeout 900 python scripts/tune_switch.py --iters 12 --repeat 2 kernel=fc kernel=fc,fc_stages=3,fc_bbufs=2,fc_astages=3 2>&1 | tail -4
