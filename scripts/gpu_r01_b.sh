#!/bin/bash
# Round-1 evidence run B: TP shard tests, MMA issue microbench, sweep, 7B drift
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_tp_shards.py -q 2>&1 | tail -4
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/mmabench2 scripts/mmabench2.cu && timeout 60 /tmp/mmabench2 | tee gpurun_out/mmabench2.txt
timeout 1500 python scripts/sweep_bench.py --out gpurun_out/r01_sweep.json 2>&1 | tail -30
timeout 1500 python scripts/drift_report.py --config llama2-7b --tokens 1000 --out gpurun_out/r01_drift_7b.json 2>&1 | tail -15
