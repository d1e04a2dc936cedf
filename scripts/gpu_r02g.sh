#!/bin/bash
mkdir -p gpurun_out
python paper_2405_17741_b200/build.py --tuning > /dev/null || exit 1
timeout 900 python scripts/fused_probe.py llama2-7b > gpurun_out/fused_probe2_7b.json 2> gpurun_out/fused_probe2_7b.err; echo "probe rc=$?"
tail -8 gpurun_out/fused_probe2_7b.err
python paper_2405_17741_b200/build.py > /dev/null || exit 1
timeout 900 python -m pytest tests/test_gpu_fused.py -q -x 2>&1 | tail -2
