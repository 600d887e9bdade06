#!/bin/bash
# End-of-round measurement pass (run under gpurun, 1 GPU): default bench line, the other configs,
# the NEXT-4 variants, ncu launch list and one full K2 capture.
mkdir -p gpurun_out
python bench.py > gpurun_out/bench_final.log 2>&1
: > gpurun_out/configs.jsonl
for cfg in "C3_hela 96" "C3_simplus 96" "C3_u373 64" "C3_gowt1 24" "C4 8"; do
  set -- $cfg
  python bench.py --config $1 --batch $2 --steps 10 --no-cpu 2>/dev/null | tail -1 >> gpurun_out/configs.jsonl
done
python bench.py --kernel-profile gauss --no-cpu --steps 10 2>/dev/null | tail -1 >> gpurun_out/configs.jsonl
python bench.py --metric euclid --no-cpu --steps 10 2>/dev/null | tail -1 >> gpurun_out/configs.jsonl
bash tools/prof.sh 96 > /dev/null 2>&1
ls -la gpurun_out
