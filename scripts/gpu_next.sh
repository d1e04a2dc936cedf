#!/bin/bash
python -c "import __graft_entry__ as g; g.build()" > /dev/null || exit 1
timeout 600 python -m pytest tests/test_gpu_fused.py -q -x 2>&1 | tail -2
for i in 1 2 3; do python scripts/fused_tune.py --lib build/liblsw_A.so llama2-7b "old:" 2>&1 | grep "^old"; python scripts/fused_tune.py llama2-7b "new:" 2>&1 | grep "^new"; done
