#!/bin/bash
# K2 wait-strategy experiments (run under gpurun): rebuild with FMS_NVCC_EXTRA, bench C2 B=32.
mkdir -p gpurun_out
for v in "" "-DFMS_WAIT_HINT" "-DK2_EPI_SLEEP=20" "-DK2_EPI_SLEEP=100" "-DK2_ROLE_SLEEP=20"; do
  FMS_NVCC_EXTRA="$v" python -c "from paper_2007_14283_b200 import build; build.build(force=True)" > /dev/null 2>&1
  r=$(python bench.py --no-cpu --no-e2e --steps 10 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],1), round(d['roofline']['achieved'],1))")
  echo "variant [$v]: frames/s, K2 TFLOP/s = $r" | tee -a gpurun_out/variants_k2.log
done
python -c "from paper_2007_14283_b200 import build; build.build(force=True)" > /dev/null 2>&1
