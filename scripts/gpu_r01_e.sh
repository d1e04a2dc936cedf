#!/bin/bash
timeout 300 python scripts/tune_gemv.py 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('math', d['groups_gemv_ms'], d['groups_gemv_GBps'], d['token_gemv_ms'])"
LSW_GEMV_PROBE=1 timeout 300 python scripts/tune_gemv.py 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('stream-only', d['groups_gemv_ms'], d['groups_gemv_GBps'], d['token_gemv_ms'])"
