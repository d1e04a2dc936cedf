#!/bin/bash
timeout 900 python -m pytest tests/test_gpu_restore.py -q -x 2>&1 | tail -2
timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print({k: d[k] for k in ['value','ms_per_step','switch_ms','restore_ms','launch_ablation','unmerged_decode_ms_per_token']})"
