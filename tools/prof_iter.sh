#!/bin/bash
# full ncu capture of a few K2 launches in steady state (run under gpurun)
mkdir -p gpurun_out
timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:iter_kernel -s 60 -c 3 \
  -o gpurun_out/prof_iter python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu --batch 32 > gpurun_out/prof_iter.log 2>&1
timeout -s KILL 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
  python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu --batch 32 > gpurun_out/launches_bench.log 2>&1
ls -la gpurun_out
