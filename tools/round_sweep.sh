#!/bin/bash
# End-of-round measurement pass (run under gpurun, 1 GPU): the default bench line (cpu baseline,
# latency, B = 16 and e2e included), the other configs, the NEXT-4 variants, the ncu launch list of
# one bench step and full captures of K2 (iter8_kernel) and K5 (assign_tc_kernel).
# Usage: tools/round_sweep.sh <tag>     (outputs gpurun_out/*_<tag>.*)
T=${1:-r02}
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/bench_$T.log 2>&1
: > gpurun_out/configs_$T.jsonl
for cfg in "C3_hela 96" "C3_simplus 96" "C3_u373 64" "C3_gowt1 24" "C4 8"; do
  set -- $cfg
  timeout 300 python bench.py --config $1 --batch $2 --steps 10 --no-cpu 2>/dev/null | tail -1 >> gpurun_out/configs_$T.jsonl
done
timeout 300 python bench.py --kernel-profile gauss --no-cpu --steps 10 2>/dev/null | tail -1 >> gpurun_out/configs_$T.jsonl
timeout 300 python bench.py --metric euclid --no-cpu --steps 10 2>/dev/null | tail -1 >> gpurun_out/configs_$T.jsonl
timeout -s KILL 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  --csv --log-file gpurun_out/launches_$T.csv python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu > /dev/null 2>&1
timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:iter8_kernel -s 40 -c 1 \
  -f -o gpurun_out/k2_$T python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu > /dev/null 2>&1
timeout -s KILL 900 ncu --set full --clock-control none -k regex:assign_tc_kernel -s 6 -c 1 \
  -f -o gpurun_out/k5_$T python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu > /dev/null 2>&1
for r in k2_$T k5_$T; do ncu -i gpurun_out/$r.ncu-rep --page raw --csv > gpurun_out/$r.raw.csv 2>/dev/null; done
ls -la gpurun_out | tail -20
