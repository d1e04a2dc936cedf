#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null || exit 1
for c in llama2-7b mistral-7b llama2-13b; do
  timeout 900 python scripts/drift_report.py --config $c --tokens 1000 --out gpurun_out/drift_$c.json > /dev/null 2> gpurun_out/drift_$c.err; echo "drift $c rc=$?"
done
SAN_ARGS= bash scripts/gpu_sanitize.sh
