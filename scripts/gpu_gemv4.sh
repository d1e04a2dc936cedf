#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_gemv4.log 2>&1 || tail -20 gpurun_out/build_gemv4.log
timeout 900 python -m pytest tests -q -m gpu -x -k "gemv or decode" 2>&1 | tail -2
for i in 1 2; do for env in "" "LSW_GEMV_NO_PREFETCH=1"; do
  env $env python scripts/tune_gemv.py 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['env'], d['groups_gemv_ms'], d['token_gemv_ms'])"
  env $env python scripts/time_fused.py 2>&1 | tail -1
done; done
