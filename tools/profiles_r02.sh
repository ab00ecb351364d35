#!/bin/bash
# round-2 evidence: ncu launch list of a short bench command, ncu --set full of a5 and of the
# fused select in the 8B-16K step, each after the same command exited 0 without ncu.
set -x
out=gpurun_out/prof2
mkdir -p $out
B="python bench.py --steps 20 --warmup 5 --no-c3 --no-heads --no-loop --no-cpu-baseline"
$B > $out/plain_bench.json 2>$out/plain_bench.err && \
  ncu --metrics gpu__time_duration.sum --clock-control none -k regex:zoomr -c 300 --csv \
      --log-file $out/launches.csv $B > $out/ncu_bench.log 2>&1
python tools/step_once.py > $out/plain_step.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:sparse_attn -s 4 -c 1 -o $out/a5 \
      python tools/step_once.py > $out/ncu_a5.log 2>&1
python tools/step_once.py > $out/plain_step2.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:fused_select -s 4 -c 1 -o $out/sel \
      python tools/step_once.py > $out/ncu_sel.log 2>&1
WL=qwen7b16k python tools/step_once.py > $out/plain_q.log 2>&1 && \
  WL=qwen7b16k ncu --set full --clock-control none --import-source on -k regex:sparse_attn -s 4 -c 1 -o $out/a5_qwen \
      python tools/step_once.py > $out/ncu_a5q.log 2>&1
echo done
