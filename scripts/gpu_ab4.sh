#!/bin/bash
mkdir -p gpurun_out
T="python scripts/tune_switch.py --iters 12"
for i in 1 2; do
echo "new"; $T kernel=fc 2>&1 | tail -1
echo "prev"; $T --lib paper_2405_17741_b200/liblsw_prev.so kernel=fc 2>&1 | tail -1
done
echo "r16k4 new"; $T --rank 16 --topk 4 --layers 16 kernel=fc 2>&1 | tail -1
echo "r16k4 prev"; $T --rank 16 --topk 4 --layers 16 --lib paper_2405_17741_b200/liblsw_prev.so kernel=fc 2>&1 | tail -1
