# prefill: parity tests, then per-group timing (auto / forced token tiles)
cd $GRAFT_REPO_ROOT
timeout 300 python -m pytest tests/test_gpu_prefill.py -q -x 2>&1 | tail -3

timeout 300 python scripts/prefill_bench.py llama2-7b 512 | python -c "
import json,sys; d=json.load(sys.stdin)
for k,v in d.items():
  if isinstance(v,dict): print(k, {g:round(x['ms']*1e3,1) for g,x in v.items()})
  elif 'layer' in k: print(k, v)"
