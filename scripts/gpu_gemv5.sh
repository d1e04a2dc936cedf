#!/bin/bash
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for i in 1 2; do for kb in 220 176 144 112; do
  LSW_GEMV_SMEM_KB=$kb python scripts/tune_gemv.py 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['env'], d['groups_gemv_ms'], d['token_gemv_ms'])"
done; done
