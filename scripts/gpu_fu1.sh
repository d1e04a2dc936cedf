#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_fu1.log 2>&1 || tail -20 gpurun_out/build_fu1.log
timeout 900 python -m pytest tests/test_gpu_fused.py -q -m gpu -x 2>&1 | tail -15
timeout 600 python scripts/time_fused.py 2>&1 | tail -3

timeout 900 python scripts/tune_switch.py --iters 12 --repeat 2 kernel=fc 2>&1 | tail -2
