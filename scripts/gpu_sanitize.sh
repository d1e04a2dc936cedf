#!/bin/bash
# compute-sanitizer over scripts/sanitize_driver.py, one tool at a time;
# summaries -> gpurun_out/sanitize_<tool>.txt
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" || exit 1
for tool in memcheck racecheck synccheck initcheck; do
  extra=""
  [ "$tool" = "racecheck" ] && extra="--racecheck-report all"
  timeout 1200 compute-sanitizer --tool $tool $extra --print-limit 50 --error-exitcode 9 \
      python scripts/sanitize_driver.py ${SAN_ARGS} > gpurun_out/sanitize_$tool.txt 2>&1
  echo "$tool rc=$?"
  tail -4 gpurun_out/sanitize_$tool.txt
done
