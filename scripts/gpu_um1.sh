#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_um1.log 2>&1 || tail -20 gpurun_out/build_um1.log
timeout 900 python -m pytest tests/test_gpu_unmerged.py tests/test_gpu_parity.py -q -m gpu -x -k "unmerged or gemv or decode" 2>&1 | tail -3
timeout 600 python scripts/time_unmerged.py 2>&1 | tail -3
