#!/bin/bash
# ncu --set full capture of one K2 (iter8_kernel) launch: in the steady-state probe (full tiles) and
# inside bench.py (the real step mix), plus the raw metric dumps (run under gpurun)
mkdir -p gpurun_out
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -Ipaper_2007_14283_b200/csrc -Iinclude \
  -o tools/iter8_probe tools/iter8_probe.cu paper_2007_14283_b200/csrc/k_iter8.cu paper_2007_14283_b200/csrc/k_iter.cu -lcuda
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:iter8_kernel -s 3 -c 1 \
  -f -o gpurun_out/prof_k2_probe ./tools/iter8_probe 32 2 64 > gpurun_out/prof_k2_probe.log 2>&1
timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:iter8_kernel -s 40 -c 1 \
  -f -o gpurun_out/prof_k2_bench python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu --batch 96 > gpurun_out/prof_k2_bench.log 2>&1
for r in prof_k2_probe prof_k2_bench; do
  ncu -i gpurun_out/$r.ncu-rep --page raw --csv > gpurun_out/$r.raw.csv 2>/dev/null
done
ls -la gpurun_out/*.ncu-rep
