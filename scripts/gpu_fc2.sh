#!/bin/bash
# fc as the default: full GPU suite, then the r=64 / N=4,16 cells
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_fc2.log 2>&1 || tail -20 gpurun_out/build_fc2.log
timeout 2400 python -m pytest tests -q -m gpu -x 2>&1 | tee gpurun_out/gpu_tests_fc2.log | tail -15
timeout 900 python scripts/sweep_bench.py --experts 8 --ranks 8,64 --topk 1,2 --out gpurun_out/sweep_fc2_def.json 2>&1 | grep -v "^{" | tail -5
