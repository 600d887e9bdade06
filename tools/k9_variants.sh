#!/bin/bash
# K2 v3 part-switch sweep (run under gpurun): iter9 cycles per tile with parts switched off (K9_OFF bits:
# 1 MMA2, 2 MMA1, 4 C loads, 8 weight stores, 16 TMA loads), then one finer timeline.
# Usage: tools/k9_variants.sh "<flags>;<flags>;..." [probe args]
set -u
SRC="tools/iter8_probe.cu paper_2007_14283_b200/csrc/k_iter8.cu paper_2007_14283_b200/csrc/k_iter.cu tools/experiments/k_iter9.cu"
F="-gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -Ipaper_2007_14283_b200/csrc -Iinclude"
IFS=';' read -ra VARS <<< "${1:-}"
shift || true
i=0
for v in "${VARS[@]:-}"; do
  nvcc $F $v -o tools/k9v$i $SRC -lcuda > /dev/null 2>&1 || { echo "build failed: [$v]"; continue; }
  echo "== variant [$v]"
  timeout 60 tools/k9v$i "$@" | grep -v "^barriers\|^iter  "
  i=$((i+1))
done
