#!/bin/bash
# configs[4] stress grid: c in {2,8,32} x L_R in {64,256,1024} x U in {1,16,64}; one bench line per point.
out=${1:-gpurun_out/stress.jsonl}
: > $out
for LR in 64 256 1024; do for c in 2 8 32; do for U in 1 16 64; do
  steps=$(( U > 16 ? 128 : 64 ))
  timeout -s KILL 300 python bench.py --steps $steps --warmup $U --rotate 2 --no-cpu-baseline --no-loop --no-c3 --no-heads --workload stress_LR${LR}_c${c}_U${U} 2>/dev/null | tail -1 >> $out
done; done; done
