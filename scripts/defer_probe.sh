cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python scripts/fused_tune.py llama2-7b "head:" > gpurun_out/fused_head.json 2>&1
timeout 300 python scripts/tune_switch.py --config llama2-7b --iters 12 --repeat 2 "" >> gpurun_out/fused_head.json 2>&1
