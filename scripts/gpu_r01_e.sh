#!/bin/bash
timeout 300 python scripts/tune_gemv.py 2>&1 | tail -1 | cut -c1-330
LSW_GEMV_SMEM_KB=200 timeout 300 python scripts/tune_gemv.py 2>&1 | tail -1 | cut -c1-330
