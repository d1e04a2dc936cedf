#!/bin/bash
# folded-coefficient kernel: parity (-k fc) then sweep cells fc vs default on the same box
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_fc1.log 2>&1 || tail -20 gpurun_out/build_fc1.log
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_restore.py -q -m gpu -k "fc" -x 2>&1 | tail -15
LSW_TC_KERNEL=fc timeout 900 python scripts/sweep_bench.py --experts 8 --ranks 4,16,32 --topk 1,2,3,4 --out gpurun_out/sweep_fc1_fc.json 2>&1 | grep -v "^{" | tail -5
timeout 900 python scripts/sweep_bench.py --experts 8 --ranks 4,16,32 --topk 1,2,3,4 --out gpurun_out/sweep_fc1_def.json 2>&1 | grep -v "^{" | tail -5
