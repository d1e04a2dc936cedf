#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_13b.log 2>&1 || tail -20 gpurun_out/build_13b.log
for L in 10 20 40; do echo "13b L=$L"; python scripts/tune_switch.py --iters 8 --config llama2-13b --layers $L kernel=fc kernel=fc,fc_pt=1 kernel=fc,probe=1 2>&1 | grep setting; done
for L in 8 32; do echo "7b L=$L"; python scripts/tune_switch.py --iters 8 --layers $L kernel=fc kernel=fc,probe=1 2>&1 | grep setting; done
