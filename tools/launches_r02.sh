#!/bin/bash
# ncu launch list (device time per launch) of the default bench's main timed part: libzoomr kernels only
mkdir -p gpurun_out/prof2
B="python bench.py --steps 20 --warmup 5 --no-c3 --no-heads --no-loop --no-cpu-baseline"
$B > gpurun_out/prof2/plain_bench2.json 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none \
    -k regex:"sparse_attn|fused_select|select_topc|score_kernel|mean_keys|build_index|zero_i64" -c 120 --csv \
    --log-file gpurun_out/prof2/launches.csv $B > gpurun_out/prof2/ncu_bench2.log 2>&1
echo rc=$?
