#!/bin/bash
timeout 600 python scripts/time_unmerged.py
LSW_UNMERGED_PREFETCH=0 timeout 600 python scripts/time_unmerged.py
timeout 600 python -m pytest tests/test_gpu_unmerged.py -q -x 2>&1 | tail -1
