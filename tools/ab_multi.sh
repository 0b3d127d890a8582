#!/bin/bash
# tools/ab_multi.sh "<workloads>" lib lib_v1 ...: kernel-only A/B over several workloads
set -u
WS=$1; shift
L=paper_2508_07071_b200/lib
cp $L/libfk_cuda.so /tmp/lib_main.so
for W in $WS; do for rep in 1 2; do for v in "$@"; do
  if [ "$v" = lib ]; then cp /tmp/lib_main.so $L/libfk_cuda.so; else cp paper_2508_07071_b200/$v/libfk_cuda.so $L/libfk_cuda.so; fi
  echo -n "$W $v "; timeout 300 python bench.py --workload $W --steps 50 --warmup 5 --no-cpu --no-e2e --no-unfused --no-sub --no-gate ${BENCH_ARGS:-} 2>/dev/null | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["ms_per_step"]*1000,2), "us frac", round(d["roofline"]["frac"],3), d["roofline"]["kernel"])'
done; done; done
cp /tmp/lib_main.so $L/libfk_cuda.so
