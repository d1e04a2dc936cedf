#!/bin/bash
# evidence run: full GPU tests, bench (3 configs), sweep, drift, launch list, ncu of switch + GEMV
mkdir -p gpurun_out
TAG=${TAG:-r01z}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_${TAG}.log 2>&1 || tail -20 gpurun_out/build_${TAG}.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 2400 python -m pytest tests -q -m gpu 2>&1 | tee gpurun_out/gpu_tests_${TAG}.log | tail -3
timeout 900 python bench.py --steps 20 --warmup 5 2>&1 | tail -1 | tee gpurun_out/bench_${TAG}.json
timeout 900 python bench.py --steps 10 --warmup 3 --config mistral-7b --no-cpu-baseline 2>&1 | tail -1 > gpurun_out/bench_${TAG}_mistral.json
timeout 900 python bench.py --steps 10 --warmup 3 --config llama2-13b --no-cpu-baseline 2>&1 | tail -1 > gpurun_out/bench_${TAG}_13b.json


timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"switch|gemv|router" -s 390 -c 260 --csv \
  --log-file gpurun_out/launches_${TAG}.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch_${TAG}.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:switch_ -s 1 -c 1 \
  -o gpurun_out/switch_${TAG} python scripts/prof_kernels.py --layers 4 --tokens 3 > gpurun_out/ncu_switch_${TAG}.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemv -s 4 -c 4 \
  -o gpurun_out/gemv_${TAG} python scripts/prof_kernels.py --layers 4 --tokens 3 > gpurun_out/ncu_gemv_${TAG}.log 2>&1
