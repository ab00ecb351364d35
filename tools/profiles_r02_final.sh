#!/bin/bash
# end-of-round-2 evidence on the final build: the ncu launch list of the default bench's main timed
# part, and ncu --set full of a5 and of the fused select in the 8B-16K step (and a5 at Qwen-7B-16K),
# each after the same command exited 0 without ncu.
out=gpurun_out/prof_final
mkdir -p $out
B="python bench.py --steps 20 --warmup 5 --no-c3 --no-heads --no-loop --no-cpu-baseline"
$B > $out/plain_bench.json 2>$out/plain_bench.err && \
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none \
      -k regex:"sparse_attn|fused_select|select_topc|score_kernel|mean_keys|build_index|zero_i64" -c 120 --csv \
      --log-file $out/launches.csv $B > $out/ncu_bench.log 2>&1
echo "launches rc=$?"
python tools/step_once.py > $out/plain_step.log 2>&1 && \
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:sparse_attn -s 4 -c 1 -o $out/a5 \
      python tools/step_once.py > $out/ncu_a5.log 2>&1
echo "a5 rc=$?"
python tools/step_once.py > $out/plain_step2.log 2>&1 && \
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:fused_select -s 4 -c 1 -o $out/sel \
      python tools/step_once.py > $out/ncu_sel.log 2>&1
echo "sel rc=$?"
WL=qwen7b16k python tools/step_once.py > $out/plain_q.log 2>&1 && \
  WL=qwen7b16k timeout 600 ncu --set full --clock-control none --import-source on -k regex:sparse_attn -s 4 -c 1 \
      -o $out/a5_qwen python tools/step_once.py > $out/ncu_a5q.log 2>&1
echo "a5q rc=$?"
for r in a5 sel a5_qwen; do
  [ -f $out/$r.ncu-rep ] && ncu -i $out/$r.ncu-rep --page raw --csv > $out/${r}_details.csv 2>/dev/null
done
echo done
