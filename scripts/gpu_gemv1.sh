#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_gemv1.log 2>&1 || tail -20 gpurun_out/build_gemv1.log
for i in 1 2; do
python scripts/tune_gemv.py 2>&1 | tail -1
LSW_GEMV_XF32=1 python scripts/tune_gemv.py 2>&1 | tail -1
done
LSW_GEMV_PROBE=1 python scripts/tune_gemv.py 2>&1 | tail -1
timeout 900 python -m pytest tests -q -m gpu -x -k "gemv or decode or unmerged or fullsize" 2>&1 | tail -3
