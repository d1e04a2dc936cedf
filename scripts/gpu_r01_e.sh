#!/bin/bash
for c in 1 2; do LSW_TC_FUSED_CHUNK=$c timeout 600 python scripts/time_fused.py; done
