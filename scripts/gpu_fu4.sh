#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_fu4.log 2>&1 || tail -20 gpurun_out/build_fu4.log
for f in 0 4 8 12; do LSW_FC_FUSED_PROBE=$f timeout 600 python scripts/time_fused.py 2>&1 | tail -1; done
timeout 900 python scripts/tune_switch.py --iters 12 --repeat 2 kernel=fc kernel=fc,probe=1 2>&1 | tail -4
timeout 900 python scripts/sweep_bench.py --experts 8 --ranks 4,16,32,64 --topk 1,2,3,4 --out gpurun_out/sweep_fu4.json 2>&1 | tail -1
