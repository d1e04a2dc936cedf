#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 900 python -m pytest tests/test_gpu_prefill.py -q -x > gpurun_out/r02c_prefill.log 2>&1; echo "prefill tests rc=$?"
tail -30 gpurun_out/r02c_prefill.log | grep -v "^$" | tail -25
for tool in racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 20 --error-exitcode 9 python scripts/sanitize_driver.py --quick > gpurun_out/sanitize_$tool.txt 2>&1
  echo "$tool rc=$?"; tail -2 gpurun_out/sanitize_$tool.txt
done
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench_r02c.json 2> gpurun_out/bench_r02c.err; echo "bench rc=$?"
python -c "
import json; d=json.loads(open('gpurun_out/bench_r02c.json').read().strip().splitlines()[-1])
print({k: d.get(k) for k in ['ms_per_step','switch_ms','gemv_ms_per_token','fused_decode_ms_per_token','prefill']})"
tail -5 gpurun_out/bench_r02c.err
