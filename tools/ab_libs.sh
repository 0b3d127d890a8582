#!/bin/bash
# A/B/..: kernel-only bench of one workload with each library variant, alternated
#   tools/ab_libs.sh <workload> lib lib_v1 lib_v2 ...   (dirs under paper_2508_07071_b200/; "lib" = the main build)
set -u
W=$1; shift
L=paper_2508_07071_b200/lib
cp $L/libfk_cuda.so /tmp/lib_main.so
for rep in 1 2; do
  for v in "$@"; do
    if [ "$v" = lib ]; then cp /tmp/lib_main.so $L/libfk_cuda.so; else cp paper_2508_07071_b200/$v/libfk_cuda.so $L/libfk_cuda.so; fi
    echo -n "$v "; timeout 300 python bench.py --workload $W --steps 20 --warmup 3 --no-cpu --no-e2e --no-unfused --no-sub --no-gate 2>/dev/null | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["ms_per_step"],4), "ms frac", round(d["roofline"]["frac"],3), d["roofline"]["kernel"])'
  done
done
cp /tmp/lib_main.so $L/libfk_cuda.so
