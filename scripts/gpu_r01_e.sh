#!/bin/bash
for cfg in "1 220" "2 110" "2 100" "3 72"; do set -- $cfg; LSW_GEMV_CTAS_PER_SM=$1 LSW_GEMV_SMEM_KB=$2 timeout 300 python scripts/tune_gemv.py 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('cps $1 smem $2', d['groups_gemv_ms'], d['token_gemv_ms'], d['token_gemv_GBps'])"; done
