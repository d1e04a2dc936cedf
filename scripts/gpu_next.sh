#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null || exit 1
timeout 900 python -m pytest tests/test_gpu_prefill.py -q -x > gpurun_out/r02p_prefill.log 2>&1; echo "prefill tests rc=$?"; tail -15 gpurun_out/r02p_prefill.log
timeout 600 python scripts/prefill_bench.py llama2-7b 512 > gpurun_out/prefill_bench_pdl.json 2>&1; echo "pb rc=$?"
python -c "
import json; d=json.load(open('gpurun_out/prefill_bench_pdl.json'))
for k in ('tt128','tt256'): print(k, d[k+'_layer_ms'], {g:round(v['ms']*1000,1) for g,v in d[k].items()})
print('torch', d['torch_dense_layer_ms'])"
