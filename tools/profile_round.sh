#!/bin/bash
# Profiling pass for profiles/ (run on the GPU box from the repo root):
#   1. the bench command alone (must exit 0 before any ncu run),
#   2. its ncu launch list (gpu__time_duration.sum, --clock-control none),
#   3. one --set full capture of the dominant kernels per config.
set -u
mkdir -p gpurun_out/prof
for c in 3 1; do
  timeout 600 python bench.py --config $c --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/prof/bench_c$c.log 2>&1 || exit 1
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 700 --csv \
    --log-file gpurun_out/prof/launches_c$c.csv \
    python bench.py --config $c --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/prof/ncu_launch_c$c.log 2>&1
  timeout 900 ncu --set full --import-source on --clock-control none \
    -k regex:"fc_tma_kernel|fr_tma_kernel|expand_diff" -c 6 -o gpurun_out/prof/full_c$c \
    python tools/one_step.py --config $c --warm 0 --synth > gpurun_out/prof/ncu_full_c$c.log 2>&1
done
ls -la gpurun_out/prof
