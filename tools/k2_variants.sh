#!/bin/bash
# K2 probe sweep (run under gpurun): build tools/iter8_probe with compile-time variants and time them.
# Usage: tools/k2_variants.sh "<nvcc -D flags>;<flags>;..." [probe args]
set -u
SRC="tools/iter8_probe.cu paper_2007_14283_b200/csrc/k_iter8.cu paper_2007_14283_b200/csrc/k_iter.cu tools/experiments/k_iter9.cu"
IFS=';' read -ra VARS <<< "${1:-}"
shift || true
i=0
for v in "${VARS[@]:-}"; do
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -Ipaper_2007_14283_b200/csrc -Iinclude \
    $v -o tools/iter8_probe_v$i $SRC -lcuda > /dev/null 2>&1 || { echo "build failed: [$v]"; continue; }
  echo "== variant [$v]"
  timeout 60 tools/iter8_probe_v$i "$@"
  i=$((i+1))
done
