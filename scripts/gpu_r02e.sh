#!/bin/bash
mkdir -p gpurun_out
python paper_2405_17741_b200/build.py --tuning > /dev/null || exit 1
timeout 900 python scripts/fused_probe.py llama2-7b > gpurun_out/fused_probe_7b.json 2> gpurun_out/fused_probe_7b.err; echo "probe rc=$?"
cat gpurun_out/fused_probe_7b.err | tail -10
python paper_2405_17741_b200/build.py > /dev/null || exit 1
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench_r02e.json 2> gpurun_out/bench_r02e.err; echo "bench rc=$?"
python -c "
import json; d=json.loads(open('gpurun_out/bench_r02e.json').read().strip().splitlines()[-1])
print({k: d.get(k) for k in ['ms_per_step','switch_ms','gemv_ms_per_token','fused_decode_ms_per_token','prefill']})"
