timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fused.py tests/test_gpu_graph.py -x -q 2>&1 | tail -1
python scripts/fused_tune.py --lib build/liblsw_pre_tb.so llama2-7b "pre:" 2>&1 | grep "^pre"
python scripts/fused_tune.py llama2-7b "now:" 2>&1 | grep "^now"
for c in llama2-7b llama2-13b; do python scripts/tune_switch.py --config $c --iters 16 --repeat 2 ""; python scripts/tune_switch.py --lib build/liblsw_pre_tb.so --config $c --iters 16 --repeat 2 ""; done
