#!/bin/bash
# timing of K2 with parts switched off (results invalid for variants != 0); run under gpurun
for v in 0 1 2 4 3 7; do
  echo -n "variant $v: "
  FMS_ITER_VARIANT=$v timeout -s KILL 300 python bench.py --steps 6 --warmup 2 --no-cpu --no-e2e --batch 16 > gpurun_out/var$v.log 2>&1; tail -2 gpurun_out/var$v.log | head -1 | cut -c1-300
  FMS_ITER_VARIANT=$v timeout -s KILL 300 python bench.py --steps 6 --warmup 2 --no-cpu --no-e2e --batch 16 2>&1 | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print(round(d['value'],1), 'fps; iter', round(r['achieved'],1), 'TF; ms/launch', round(r['ms_per_launch'],4), 'share', round(r['iter_share_of_step'],2), 'seed_iters/frame', round(d['seed_iters_per_frame']))"
done
