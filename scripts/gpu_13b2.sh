#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_13b2.log 2>&1 || tail -20 gpurun_out/build_13b2.log
echo "13b L40"; python scripts/tune_switch.py --iters 16 --config llama2-13b kernel=fc kernel=fc,chunk=96 kernel=fc,chunk=192 kernel=fc,probe=1 2>&1 | grep setting
echo "13b L30"; python scripts/tune_switch.py --iters 16 --config llama2-13b --layers 30 kernel=fc 2>&1 | grep setting
echo "7b r32 L32"; python scripts/tune_switch.py --iters 16 --rank 32 kernel=fc 2>&1 | grep setting
