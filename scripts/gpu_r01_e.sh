#!/bin/bash
python scripts/tune_switch.py --repeat 2 "order=sweep" "l2promo=0" "l2promo=128" "wpolicy=normal" "probe=1" "probe=1,l2promo=0" "probe=1,wpolicy=normal" 2>&1 | grep setting
