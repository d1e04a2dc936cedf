#!/bin/bash
# fc tuning on the 7B shape (full 32 layers)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_fc3.log 2>&1 || tail -20 gpurun_out/build_fc3.log
timeout 1200 python scripts/tune_switch.py --iters 12 --repeat 2 kernel=v1 kernel=fc kernel=fc,fc_astages=2 kernel=fc,fc_astages=2,fc_bbufs=2 \
  kernel=fc,fc_stages=3 kernel=fc,chunk=32 kernel=fc,chunk=96 kernel=fc,fc_astages=2,chunk=96 kernel=fc,probe=1 kernel=fc,probe=1,fc_astages=2 2>&1 | tee gpurun_out/tune_fc3.txt | tail -24
