# prefill: parity tests, then per-group timing (auto / forced token tiles) twice
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_prefill.py tests/test_gpu_fullsize.py -q -x -k "prefill" 2>&1 | tail -3
