#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_e2e.log 2>&1 || tail -20 gpurun_out/build_e2e.log
timeout 900 python -m pytest tests -q -m gpu -x -k "host or decode_token" 2>&1 | tail -2
timeout 900 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-restore 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['e2e'])"
