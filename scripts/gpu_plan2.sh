#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_plan2.log 2>&1 || tail -20 gpurun_out/build_plan2.log
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "many_tiles" 2>&1 | tail -2
T="python scripts/tune_switch.py --iters 8 --layers 16"
echo "r16k2 new vs old"; $T --rank 16 --topk 2 kernel=fc kernel=fc,fc_stages=3,fc_bbufs=2,fc_astages=3 kernel=fc 2>&1 | grep setting
echo "r16k3"; $T --rank 16 --topk 3 kernel=fc kernel=fc,fc_stages=4,fc_bbufs=1,fc_astages=2 2>&1 | grep setting
echo "r16k4"; $T --rank 16 --topk 4 kernel=fc kernel=fc,fc_stages=3,fc_bbufs=1,fc_astages=2 2>&1 | grep setting
echo "r32k3 pt"; $T --rank 32 --topk 3 kernel=fc kernel=fc,fc_stages=3,fc_bbufs=2,fc_astages=2 2>&1 | grep setting
echo "r32k4 pt"; $T --rank 32 --topk 4 kernel=fc kernel=fc,fc_stages=4,fc_bbufs=1,fc_astages=2 2>&1 | grep setting
echo "r64k1 pt"; $T --rank 64 --topk 1 kernel=fc kernel=fc,fc_stages=3,fc_bbufs=2,fc_astages=2 2>&1 | grep setting
echo "r64k2 pt"; $T --rank 64 --topk 2 kernel=fc 2>&1 | grep setting
echo "r64k3 pt"; $T --rank 64 --topk 3 kernel=fc 2>&1 | grep setting
echo "13b"; python scripts/tune_switch.py --iters 8 --config llama2-13b --layers 20 kernel=fc 2>&1 | grep setting
