#!/bin/bash
# ncu capture (full set + source) of one K2 launch inside tools/iter_probe (run under gpurun)
mkdir -p gpurun_out
B=${1:-iter_probe_h0}
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:iter_kernel -s 4 -c 1 \
  -o gpurun_out/prof_probe ./tools/$B 8 2 0 256 > gpurun_out/prof_probe.log 2>&1
tail -3 gpurun_out/prof_probe.log
