#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 600 python scripts/prefill_bench.py llama2-7b 512 > gpurun_out/prefill_bench_7b.json 2>&1; echo "pb rc=$?"
cat gpurun_out/prefill_bench_7b.json | python -c "import json,sys; d=json.load(sys.stdin); print({k:v for k,v in d.items() if 'ms' in k})"
timeout 600 python -m pytest tests/test_gpu_prefill.py -q -x > gpurun_out/r02d_prefill.log 2>&1; echo "prefill tests rc=$?"; tail -2 gpurun_out/r02d_prefill.log
timeout 900 compute-sanitizer --tool racecheck --print-limit 20 --error-exitcode 9 python scripts/sanitize_driver.py --quick > gpurun_out/sanitize_racecheck.txt 2>&1
echo "racecheck rc=$?"; tail -2 gpurun_out/sanitize_racecheck.txt
