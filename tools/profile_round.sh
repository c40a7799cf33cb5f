#!/bin/bash
# Profiling pass for profiles/ (run on the GPU box from the repo root):
#   1. the bench line of every BASELINE config (plain runs, no profiler),
#   2. ncu launch lists of the bench command (gpu__time_duration.sum,
#      --clock-control none) for configs 3, 1 and 5,
#   3. one --set full capture of the dominant kernels of configs 3, 1 and 5
#      (summarised on the box), 4. CUPTI kernel timelines of configs 5, 3, 1.
# Each ncu command runs only after the same command exited 0 without ncu.
set -u
mkdir -p gpurun_out/prof
for c in 3 1 2 4 5; do
  timeout 900 python bench.py --config $c > gpurun_out/prof/bench_c$c.json 2> gpurun_out/prof/bench_c$c.err || exit 1
done
for c in 3 1 5; do
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 1000 --csv \
    --log-file gpurun_out/prof/launches_c$c.csv \
    python bench.py --config $c --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/prof/ncu_launch_c$c.log 2>&1
done
for c in 3 1 5; do
  # reports stay on the box (gpurun_out is capped at 64 MiB); summaries come back
  timeout 900 ncu -f --set full --import-source on --clock-control none \
    -k regex:"fc_tma_kernel|fr_tma_kernel|fr_wide_kernel|expand_tma|finish_step|prep_cluster|cholqr_cluster" -c 10 -o /tmp/full_c$c \
    python tools/one_step.py --config $c --warm 0 --synth > gpurun_out/prof/ncu_full_c$c.log 2>&1
  python tools/ncu_summary.py /tmp/full_c$c.ncu-rep > gpurun_out/prof/ncu_full_c${c}_summary.txt 2>&1
  python tools/ncu_summary.py /tmp/full_c$c.ncu-rep --json > gpurun_out/prof/ncu_full_c${c}.json 2>&1
done
for c in 5 3 1; do
  timeout 300 python tools/timeline.py --config $c --gaps 10 > gpurun_out/prof/timeline_c$c.txt 2>&1
done
ls -la gpurun_out/prof
