#!/bin/bash
# A/B of the direct kernel (C1 and C3 at several chain lengths): lib (A) vs lib_alt (B)
set -u
L=paper_2508_07071_b200/lib
run() { timeout 300 python bench.py --workload $1 ${2:+--n-ops $2} --steps 20 --warmup 3 --no-cpu --no-e2e --no-unfused 2>&1 | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["ms_per_step"]*1000,1), "us", round(d["roofline"]["frac"],3))'; }
for t in A B; do
  if [ $t = B ]; then cp $L/libfk_cuda.so /tmp/libA.so; cp paper_2508_07071_b200/lib_alt/libfk_cuda.so $L/libfk_cuda.so; fi
  echo "$t c1 $(run c1)  c3/1 $(run c3 1)  c3/64 $(run c3 64)  c3/1000 $(run c3 1000)"
  if [ $t = B ]; then cp /tmp/libA.so $L/libfk_cuda.so; fi
done
