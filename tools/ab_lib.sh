#!/bin/bash
# A/B: kernel-only C5 with lib (A) and lib_alt (B)
set -u
L=paper_2508_07071_b200/lib
for t in A B A B; do
  if [ $t = B ]; then cp $L/libfk_cuda.so /tmp/libA.so; cp paper_2508_07071_b200/lib_alt/libfk_cuda.so $L/libfk_cuda.so; fi
  echo -n "$t "; timeout 300 python bench.py --workload c5 --steps 20 --warmup 3 --no-cpu --no-e2e --no-unfused 2>&1 | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["ms_per_step"], d["roofline"]["frac"])'
  if [ $t = B ]; then cp /tmp/libA.so $L/libfk_cuda.so; fi
done
