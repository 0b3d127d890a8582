#!/bin/bash
# A/B of one library under two environment settings: C5 kernel-only timings.
#   tools/ab_env.sh "FK_SEP_NOBULK=1"
set -u
run() { env $1 timeout 300 python bench.py --workload c5 --steps 20 --warmup 3 --no-cpu --no-e2e --no-unfused 2>&1 | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["ms_per_step"],4), round(d["roofline"]["frac"],3))'; }
for t in A B A B; do
  if [ $t = A ]; then echo "A (default) $(run X=1)"; else echo "B ($1) $(run "$1")"; fi
done
