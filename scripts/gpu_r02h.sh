#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null || exit 1
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fused.py tests/test_gpu_restore.py tests/test_gpu_tp_shards.py -q -x 2>&1 | tail -2
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench_r02h.json 2> gpurun_out/bench_r02h.err; echo "bench rc=$?"
python -c "
import json; d=json.loads(open('gpurun_out/bench_r02h.json').read().strip().splitlines()[-1])
print({k: d.get(k) for k in ['ms_per_step','switch_ms','switch_GBps','gemv_ms_per_token','fused_decode_ms_per_token','merge_GBps','restore_GBps']})"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:switch_fc_kernel -c 4 \
   -o gpurun_out/prof_fused2 python scripts/prof_fused.py > gpurun_out/prof_fused2.log 2>&1; echo "ncu rc=$?"
