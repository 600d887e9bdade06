#!/bin/bash
# K2 v3 (k_iter9.cu) probe pass (run under gpurun): timing + exactness vs iter8, and a timeline.
# Usage: tools/k9_probe.sh "<extra nvcc -D flags>"
set -u
mkdir -p gpurun_out
SRC="tools/iter8_probe.cu paper_2007_14283_b200/csrc/k_iter8.cu paper_2007_14283_b200/csrc/k_iter.cu tools/experiments/k_iter9.cu"
F="-gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -Ipaper_2007_14283_b200/csrc -Iinclude ${1:-}"
nvcc $F -o tools/k9p $SRC -lcuda || exit 1
nvcc $F -DK9_TIMELINE -o tools/k9pt $SRC -lcuda || exit 1
for args in "32 2 64" "32 2 32" "32 2 16" "96 1 32" "32 2 32 262144 16 160" "64 3 32 262144 16 300"; do
  echo "== probe $args"; timeout 60 tools/k9p $args
done
echo "== timeline"; timeout 60 tools/k9pt 32 2 32 | tail -45
