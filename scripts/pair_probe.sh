# switch on CTA pairs (tc_pair=1): parity, then the per-tile trace (tuning build)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "many_tiles_per_cta" > gpurun_out/pair_tests.log 2>&1; tail -2 gpurun_out/pair_tests.log
python paper_2405_17741_b200/build.py --tuning > /dev/null
timeout 300 python scripts/fused_trace.py llama2-7b 4 tc_pair=1 > gpurun_out/trace_pair.json 2>&1
timeout 300 python scripts/fused_trace.py llama2-7b 4 > gpurun_out/trace_single.json 2>&1
python paper_2405_17741_b200/build.py > /dev/null
