#!/bin/bash
mkdir -p gpurun_out
T="python scripts/tune_switch.py --iters 10 --layers 16 --repeat 2"
for rk in "16 2" "16 3" "16 4" "32 2"; do set -- $rk
echo "r$1 k$2 new"; $T --rank $1 --topk $2 kernel=fc 2>&1 | tail -2
echo "r$1 k$2 old"; $T --rank $1 --topk $2 --lib paper_2405_17741_b200/liblsw_r01s.so kernel=fc 2>&1 | tail -2
done
