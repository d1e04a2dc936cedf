#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_fc4.log 2>&1 || tail -20 gpurun_out/build_fc4.log
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "many_tiles and mini-r32" 2>&1 | tail -2
LSW_FC_WRM=1 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_restore.py -q -m gpu -x -k "many_tiles or trajectory or restore or ablation" 2>&1 | tail -2
timeout 1200 python scripts/tune_switch.py --iters 12 --repeat 3 kernel=fc kernel=fc,fc_wrm=1 kernel=fc,probe=1 kernel=fc,probe=1,fc_wrm=1 2>&1 | tee gpurun_out/tune_fc4.txt | tail -12
