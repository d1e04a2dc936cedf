#!/bin/bash
python -c "import __graft_entry__ as g; g.build()" > /dev/null || exit 1
timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "mini-r32 and tc and (test_switch_trajectory or many_tiles)" 2>&1 | tail -15
timeout 300 python scripts/tune_switch.py --config llama2-13b --repeat 2 "tc_pair=0" "tc_pair=1" 2>&1 | tail -4
