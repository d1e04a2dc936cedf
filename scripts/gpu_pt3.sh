#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_pt3.log 2>&1 || tail -20 gpurun_out/build_pt3.log
timeout 2400 python -m pytest tests -q -m gpu 2>&1 | tee gpurun_out/gpu_tests_pt3.log | tail -3
timeout 1500 python scripts/sweep_bench.py --out gpurun_out/r01_sweep_pt3.json > /dev/null 2>&1
timeout 900 python scripts/tune_switch.py --iters 12 --repeat 2 kernel=fc 2>&1 | grep setting
