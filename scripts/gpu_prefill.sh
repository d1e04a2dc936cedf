#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_pf.log 2>&1 || tail -20 gpurun_out/build_pf.log
timeout 900 python -m pytest tests/test_gpu_prefill.py -q -m gpu -x 2>&1 | tail -15
