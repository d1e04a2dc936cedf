# Unmerged decode A/B: parity tests, then decode_ab (token of GEMVs, unmerged token)
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_unmerged.py -q -x 2>&1 | tail -2
for rep in 1 2 3; do
python scripts/decode_ab.py llama2-7b 2>&1 | tail -1
done
python scripts/decode_ab.py llama2-13b 2>&1 | tail -1
python scripts/decode_ab.py mistral-7b 2>&1 | tail -1
