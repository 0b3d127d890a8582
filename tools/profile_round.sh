#!/bin/bash
# One profiling pass (run under gpurun): the launch list of the default bench
# command, one `ncu --set full` capture per workload, and the bench line itself.
#   tools/profile_round.sh <tag>
set -u
T=${1:-r01}
mkdir -p gpurun_out
B="python bench.py --steps 5 --warmup 3 --no-cpu --no-e2e --no-unfused"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/launches_${T}.csv $B > /dev/null 2>&1
for w in ${WLS:-c5 c1 c3}; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:"fk_direct|fk_resample|fk_transform" -c 1 \
    -o gpurun_out/prof_${T}_$w $B --workload $w --steps 1 > /dev/null 2>&1
done
timeout 600 python bench.py > gpurun_out/bench_${T}.json 2> gpurun_out/bench_${T}.err
ls -la gpurun_out | tail -12
