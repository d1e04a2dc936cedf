#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_plan3.log 2>&1 || tail -20 gpurun_out/build_plan3.log
T="python scripts/tune_switch.py --iters 8 --layers 16"
echo "r16k3"; $T --rank 16 --topk 3 kernel=fc kernel=fc,fc_pt=1 2>&1 | grep setting
echo "r16k4"; $T --rank 16 --topk 4 kernel=fc kernel=fc,fc_pt=1 2>&1 | grep setting
echo "r32k2"; $T --rank 32 --topk 2 kernel=fc kernel=fc,fc_pt=1 2>&1 | grep setting
echo "13b"; python scripts/tune_switch.py --iters 8 --config llama2-13b --layers 20 kernel=fc kernel=fc,fc_pt=1 2>&1 | grep setting
echo "13b L40"; python scripts/tune_switch.py --iters 8 --config llama2-13b kernel=fc kernel=fc,fc_pt=1 2>&1 | grep setting
