#!/bin/bash
# K2 work-item size experiment (run under gpurun): rebuild with -DFMS_CHUNK_TILES=c, bench C2 B=96.
mkdir -p gpurun_out
for c in 16 32 8; do
  FMS_NVCC_EXTRA="-DFMS_CHUNK_TILES=$c" python -c "from paper_2007_14283_b200 import build; build.build(force=True)" > /dev/null 2>&1
  r=$(python bench.py --no-cpu --no-e2e --steps 10 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],1), round(d['roofline']['achieved'],1))")
  echo "chunk tiles $c: frames/s, K2 TFLOP/s = $r" | tee -a gpurun_out/variants_chunk.log
done
python -c "from paper_2007_14283_b200 import build; build.build(force=True)" > /dev/null 2>&1
