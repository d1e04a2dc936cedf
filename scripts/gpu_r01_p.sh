#!/bin/bash
# round-1 re-entry check: smoke, full GPU tests, default bench on a fresh box
mkdir -p gpurun_out
TAG=${TAG:-r01p}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_${TAG}.log 2>&1 || tail -20 gpurun_out/build_${TAG}.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 2400 python -m pytest tests -q -m gpu 2>&1 | tee gpurun_out/gpu_tests_${TAG}.log | tail -3
timeout 900 python bench.py --steps 20 --warmup 5 2>&1 | tail -1 | tee gpurun_out/bench_${TAG}.json
