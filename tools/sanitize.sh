#!/bin/bash
# compute-sanitizer over tools/sanitize_driver.py (every libzoomr kernel on small
# workloads); one log per tool under profiles/ (usage: tools/sanitize.sh [outdir]).
out=${1:-profiles}
mkdir -p "$out"
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck racecheck synccheck initcheck; do
  extra=""
  [ "$tool" = "memcheck" ] && extra="--leak-check full"
  [ "$tool" = "initcheck" ] && extra="--track-unused-memory no"
  timeout 1500 $CS --tool $tool $extra --kernel-name regex:zoomr --print-limit 50 \
      python tools/sanitize_driver.py > "$out/r02_sanitizer_$tool.log" 2>&1
  echo "$tool rc=$?" >> "$out/r02_sanitizer_summary.txt"
  grep -E "ERROR SUMMARY|RACECHECK SUMMARY|LEAK SUMMARY" "$out/r02_sanitizer_$tool.log" >> "$out/r02_sanitizer_summary.txt"
done
