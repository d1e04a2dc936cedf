#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 1800 python -m pytest tests/test_gpu_router.py tests/test_gpu_nccl.py tests/test_gpu_fullsize.py -q -s -rs > gpurun_out/r02a_tests.log 2>&1; echo "tests rc=$?"
grep -E "passed|failed|worst|drift|SKIP|Error|assert" gpurun_out/r02a_tests.log | tail -30
SAN_ARGS=--quick bash scripts/gpu_sanitize.sh
