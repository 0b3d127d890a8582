#!/bin/bash
# One GPU iteration (run under gpurun): the -m gpu suite and kernel-only bench
# lines for the given workloads (full JSON lines into gpurun_out/bench_<w>.json).
#   tools/gpu_round.sh "c5 c2 c1 c3 c4" [pytest-args]
set -u
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
timeout 900 python -m pytest tests -m gpu -q -x ${2:-} 2>&1 | tail -15
for w in ${1:-c5}; do
  timeout 300 python bench.py --workload "$w" --steps 20 --warmup 3 --no-cpu --no-e2e 2>gpurun_out/bench_$w.err | tail -1 > gpurun_out/bench_$w.json
  python - "$w" <<'PY'
import json, sys
w = sys.argv[1]
l = open(f"gpurun_out/bench_{w}.json").read().strip()
try:
    d = json.loads(l); r = d["roofline"]; u = d.get("unfused") or {}
    print(w, d["config"]["workload"][:50], "| ms", round(d["ms_per_step"], 4), "GB/s", round(r["achieved"]),
          "frac", round(r["frac"], 3), "kernel", r.get("kernel"), "| unfused ms", round(u.get("ms_per_step", 0), 4))
except Exception:
    print("bench failed:", w, l[-300:], open(f"gpurun_out/bench_{w}.err").read()[-600:])
PY
done
