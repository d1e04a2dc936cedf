#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_w3.log 2>&1 || tail -20 gpurun_out/build_w3.log
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_restore.py tests/test_gpu_fused.py -q -m gpu -x 2>&1 | tail -2
for rk in "4 1" "16 1" "16 2" "32 1" "64 1"; do set -- $rk
  python scripts/tune_switch.py --iters 12 --rank $1 --topk $2 kernel=fc 2>&1 | grep setting | sed "s/^/r$1k$2 /"
done
timeout 1500 python scripts/sweep_bench.py --out gpurun_out/r01_sweep_w3.json > /dev/null 2>&1
