#!/bin/bash
# One `ncu --set full` capture of the fused kernel of a bench workload (run under gpurun):
#   tools/ncu_one.sh <workload> <regex> <tag>
set -u
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$2" -c 1 -o "gpurun_out/$3" \
  python bench.py --workload "$1" --steps 1 --warmup 3 --no-cpu --no-e2e --no-unfused > "gpurun_out/$3.log" 2>&1
tail -2 "gpurun_out/$3.log"
