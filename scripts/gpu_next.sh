#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null || exit 1
timeout 900 python -m pytest tests/test_gpu_prefill.py -q -x > gpurun_out/r02p_prefill.log 2>&1; echo "prefill tests rc=$?"; tail -3 gpurun_out/r02p_prefill.log
timeout 600 python scripts/prefill_bench.py llama2-7b 512 > gpurun_out/prefill_bench_cl.json 2>&1; echo "pb rc=$?"
python paper_2405_17741_b200/build.py --tuning > /dev/null
timeout 600 python scripts/fused_trace.py > gpurun_out/fused_trace.json 2> gpurun_out/fused_trace.err; echo "trace rc=$?"
python paper_2405_17741_b200/build.py > /dev/null
