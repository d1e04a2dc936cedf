#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_pt2.log 2>&1 || tail -20 gpurun_out/build_pt2.log
T="python scripts/tune_switch.py --iters 8 --layers 16"
for rk in "16 3" "32 3" "32 4" "64 2" "64 3" "64 4"; do set -- $rk
echo "r$1 k$2"; $T --rank $1 --topk $2 kernel=fc,fc_pt=0 kernel=fc,fc_pt=1 kernel=tg 2>&1 | grep setting
done
echo "13b"; python scripts/tune_switch.py --iters 8 --config llama2-13b --layers 20 kernel=fc,fc_pt=0 kernel=fc,fc_pt=1 2>&1 | grep setting
