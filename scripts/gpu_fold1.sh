#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "many_tiles and (mini-r32 or mini-r4k4)" 2>&1 | tail -2
P=paper_2405_17741_b200/liblsw_prev.so
echo "13b"; python scripts/tune_switch.py --iters 16 --config llama2-13b --layers 20 kernel=fc kernel=fc,probe=16 2>&1 | grep setting
python scripts/tune_switch.py --iters 16 --config llama2-13b --layers 20 --lib $P kernel=fc 2>&1 | grep setting
echo "r16k4"; python scripts/tune_switch.py --iters 16 --layers 16 --rank 16 --topk 4 kernel=fc kernel=fc,probe=16 2>&1 | grep setting
python scripts/tune_switch.py --iters 16 --layers 16 --rank 16 --topk 4 --lib $P kernel=fc 2>&1 | grep setting
echo "7b"; python scripts/tune_switch.py --iters 12 kernel=fc 2>&1 | grep setting
python scripts/tune_switch.py --iters 12 --lib $P kernel=fc 2>&1 | grep setting
