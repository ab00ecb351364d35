#!/bin/bash
# A/B of tools/probe_a5.py across library builds on one box: tools/ab_probe.sh out.jsonl lib1.so lib2.so ...
# (workloads from $WLS, default "WL=8b16k|WL=qwen7b16k|WL=70b64k HKV=1 HQ=8"; ROUNDS alternations)
out=$1; shift
IFS='|' read -ra W <<< "${WLS:-WL=8b16k|WL=qwen7b16k|WL=70b64k HKV=1 HQ=8}"
for r in $(seq 1 ${ROUNDS:-2}); do
  for w in "${W[@]}"; do
    for lib in "$@"; do
      echo -n "{\"lib\": \"$(basename $lib)\", \"round\": $r, \"probe\": " >> "$out"
      env $w ZOOMR_LIB_OVERRIDE=$(realpath $lib) python tools/probe_a5.py >> "$out" 2>>"${out%.jsonl}.err" || echo "null" >> "$out"
      echo "}" >> "$out"
    done
  done
done
