#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_fc6.log 2>&1 || tail -20 gpurun_out/build_fc6.log
T="python scripts/tune_switch.py --iters 10 --layers 16"
echo "r16 k3"; $T --rank 16 --topk 3 kernel=fc kernel=fc,fc_stages=3 kernel=fc,probe=1 2>&1 | tail -3
echo "r16 k4"; $T --rank 16 --topk 4 kernel=fc kernel=fc,probe=1 kernel=fc,chunk=24 2>&1 | tail -3
echo "r32 k2"; $T --rank 32 --topk 2 kernel=fc kernel=fc,probe=1 kernel=fc,chunk=24 kernel=fc,fc_astages=3,fc_stages=2 2>&1 | tail -4
echo "13b"; python scripts/tune_switch.py --iters 10 --config llama2-13b --layers 20 kernel=fc kernel=fc,probe=1 kernel=tg 2>&1 | tail -3
