#!/bin/bash
# Round profile pass (run under gpurun, 1 GPU): ncu launch list of one bench step, one full
# capture of K2 in steady state, and the clock record.
mkdir -p gpurun_out
B=${1:-32}
timeout -s KILL 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
  python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu --batch $B > gpurun_out/launches_bench.log 2>&1
timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:iter_kernel -s 60 -c 1 \
  -o gpurun_out/prof_iter python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu --batch $B > gpurun_out/prof_iter.log 2>&1
ls -la gpurun_out
