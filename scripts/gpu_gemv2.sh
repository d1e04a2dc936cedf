#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_gemv2.log 2>&1 || tail -20 gpurun_out/build_gemv2.log
for env in "" "LSW_GEMV_OP_KB=16" "LSW_GEMV_OP_KB=48" "LSW_GEMV_OP_KB=64" "LSW_GEMV_SMEM_KB=200" "LSW_GEMV_SMEM_KB=160" "LSW_GEMV_TOKEN=1"; do
  env $env python scripts/tune_gemv.py 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['env'], d['groups_gemv_ms'], d['token_gemv_ms'])"
done
