#!/bin/bash
# A/B on one box: a5 early-known rows (I_p, I_w before the wait) vs index-only.
set -x
VARS=late,early,late,early python tools/ab_step.py
python bench.py --steps 200 --warmup 20 --no-cpu-baseline > gpurun_out/bench_early.json 2>gpurun_out/bench_early.err
python bench.py --steps 200 --warmup 20 --no-cpu-baseline --no-early > gpurun_out/bench_late.json 2>>gpurun_out/bench_early.err
python bench.py --steps 200 --warmup 20 --no-cpu-baseline > gpurun_out/bench_early2.json 2>>gpurun_out/bench_early.err
