#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_ab3.log 2>&1 || tail -20 gpurun_out/build_ab3.log
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fused.py tests/test_gpu_restore.py -q -m gpu -x -k "many_tiles or fused or trajectory or restore" 2>&1 | tail -2
T="python scripts/tune_switch.py --iters 10 --layers 16 --repeat 2"
for rk in "16 2" "16 3" "16 4" "32 2"; do set -- $rk
echo "r$1 k$2"; $T --rank $1 --topk $2 kernel=fc 2>&1 | tail -2
done
for f in 0 8; do LSW_FC_FUSED_PROBE=$f timeout 600 python scripts/time_fused.py 2>&1 | tail -1; done
