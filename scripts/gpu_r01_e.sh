#!/bin/bash
for kb in 16 32 48 64; do LSW_GEMV_OP_KB=$kb timeout 300 python scripts/tune_gemv.py 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('op', $kb, 'groups', d['groups_gemv_ms'], d['groups_gemv_GBps'])"; done
export LSW_GEMV_TOKEN=1
for f in 0 2; do for kb in 48 96; do LSW_GEMV_TOKEN_FLAGS=$f LSW_GEMV_SLOT_KB=$kb timeout 300 python scripts/tune_gemv.py 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('token flags', $f, 'slot', $kb, d['token_gemv_ms'], d['token_gemv_GBps'])"; done; done
