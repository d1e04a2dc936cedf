#!/bin/bash
# Round evidence on one B200 (all outputs under gpurun_out/, summarised into
# profiles/ by scripts/summarize_profiles.py TAG):
#   smoke, pytest -m gpu, bench.py for the three BASELINE shapes, the ncu
#   launch list of two timed bench tokens, ncu --set full captures of the
#   switch + GEMVs (4-layer 7B slice), the fused decode and the prefill kernels,
#   and the configs[4] sweep.
TAG=${TAG:-r02}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; echo "smoke rc=$?"
timeout 2400 python -m pytest tests -m gpu -q -rs > gpurun_out/gputests_$TAG.log 2>&1; echo "gpu tests rc=$?"
tail -3 gpurun_out/gputests_$TAG.log
timeout 900 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo "bench 7b rc=$?"
for c in mistral-7b llama2-13b; do
  timeout 900 python bench.py --config $c --no-cpu-baseline > gpurun_out/bench_${TAG}_$c.json 2> gpurun_out/bench_${TAG}_$c.err; echo "bench $c rc=$?"
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"switch_fc|gemv_bulk|router_topk" \
   --launch-skip 390 -c 260 --csv --log-file gpurun_out/launches_$TAG.csv \
   python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-restore > /dev/null 2>&1; echo "launch list rc=$?"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:switch_fc --launch-skip 1 -c 1 \
   -o gpurun_out/switch_$TAG python scripts/prof_kernels.py --layers 4 --tokens 2 > /dev/null 2>&1; echo "ncu switch rc=$?"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:gemv_bulk -c 4 \
   -o gpurun_out/gemv_$TAG python scripts/prof_kernels.py --layers 4 --tokens 2 > /dev/null 2>&1; echo "ncu gemv rc=$?"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:switch_fc -c 4 \
   -o gpurun_out/fused_$TAG python scripts/prof_fused.py > /dev/null 2>&1; echo "ncu fused rc=$?"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"prefill" -c 12 \
   -o gpurun_out/prefill_$TAG python scripts/prof_prefill.py > /dev/null 2>&1; echo "ncu prefill rc=$?"
timeout 1800 python scripts/sweep_bench.py --out gpurun_out/sweep_$TAG.json > /dev/null 2> gpurun_out/sweep_$TAG.err; echo "sweep rc=$?"
timeout 600 python scripts/prefill_bench.py llama2-7b 512 > gpurun_out/prefill_bench_$TAG.json 2>&1; echo "prefill bench rc=$?"
