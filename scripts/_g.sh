timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_unmerged.py tests/test_gpu_tp_shards.py -x -q -k "gemv or decode or unmerged or shard" 2>&1 | tail -1
for i in 1 2; do for c in llama2-7b mistral-7b llama2-13b; do python scripts/decode_ab.py $c; python scripts/decode_ab.py $c gemv_op_kb=32; done; done
python scripts/gemv_groups.py llama2-7b
