#!/bin/bash
# GPU check run under gpurun: smoke, GPU parity tests.
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -20
timeout 1200 python -m pytest tests -q -m gpu -s -x ${PYTEST_ARGS} 2>&1 | tail -60
