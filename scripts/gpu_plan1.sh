#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_plan1.log 2>&1 || tail -20 gpurun_out/build_plan1.log
T="python scripts/tune_switch.py --iters 8 --layers 16"
echo "r16k4"; $T --rank 16 --topk 4 kernel=fc kernel=fc,fc_stages=2,fc_bbufs=1,fc_astages=3 2>&1 | grep setting
echo "r16k3"; $T --rank 16 --topk 3 kernel=fc kernel=fc,fc_stages=2,fc_bbufs=1,fc_astages=4 kernel=fc,fc_stages=3,fc_bbufs=1,fc_astages=3 2>&1 | grep setting
echo "r32k3 pt"; $T --rank 32 --topk 3 kernel=fc kernel=fc,fc_stages=2,fc_bbufs=1,fc_astages=7 kernel=fc,fc_stages=3,fc_bbufs=1,fc_astages=5 2>&1 | grep setting
echo "r64k2 pt"; $T --rank 64 --topk 2 kernel=fc kernel=fc,fc_stages=2,fc_bbufs=1,fc_astages=3 2>&1 | grep setting
echo "r64k3 pt"; $T --rank 64 --topk 3 kernel=fc kernel=fc,fc_stages=2,fc_bbufs=1,fc_astages=2 2>&1 | grep setting
echo "13b"; python scripts/tune_switch.py --iters 8 --config llama2-13b --layers 20 kernel=fc kernel=fc,fc_stages=2,fc_bbufs=1,fc_astages=3 2>&1 | grep setting
