#!/bin/bash
# compute-sanitizer over every kernel family (tools/sanitize_cases.py), one log per tool.
# usage (GPU box): bash tools/sanitize.sh [outdir]
out=${1:-gpurun_out}
mkdir -p "$out"
python -c "import __graft_entry__ as g; g.build()" >/dev/null
for tool in memcheck racecheck synccheck initcheck; do
  extra=""
  [ "$tool" = racecheck ] && extra="--racecheck-report hazard"
  timeout 900 compute-sanitizer --tool $tool $extra --print-limit 50 \
    python tools/sanitize_cases.py > "$out/sanit_$tool.log" 2>&1
  echo "$tool exit $?" >> "$out/sanit_summary.txt"
  grep -E "ERROR SUMMARY|RACECHECK SUMMARY|hazard|Invalid|uninitialized" "$out/sanit_$tool.log" | tail -5 >> "$out/sanit_summary.txt"
done
