#!/bin/bash
# One GPU iteration (run under gpurun): the -m gpu suite, kernel-only bench lines
# for the given workloads, and optionally one `ncu --set full` capture of C5.
#   tools/gpu_check.sh "c5 c2 c1" [prof_tag]
set -u
mkdir -p gpurun_out
timeout 500 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
for w in ${1:-c5 c2}; do
  timeout 300 python bench.py --workload "$w" --steps 20 --warmup 3 --no-cpu --no-e2e --no-unfused 2>&1 | tail -1 |
    python -c 'import json,sys
l = sys.stdin.read().strip()
try:
    d = json.loads(l); r = d["roofline"]
    print(d["config"]["workload"][:40], "ms", round(d["ms_per_step"], 4), "GB/s", round(r["achieved"]), "frac", round(r["frac"], 3))
except Exception:
    print("bench failed:", l[-400:])'
done
if [ -n "${2:-}" ]; then
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:fk_ -c 1 -o "gpurun_out/$2" \
    python bench.py --workload c5 --steps 1 --warmup 3 --no-cpu --no-e2e --no-unfused > /dev/null 2>&1
  ls gpurun_out | grep "$2"
fi
