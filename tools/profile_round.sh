#!/bin/bash
# One profiling pass (run under gpurun): the launch list of the default bench
# command, one `ncu --set full` capture per workload, summarised ON THE BOX into
# gpurun_out/profiles/ (the reports exceed gpurun's return limit; KEEP=1 keeps
# them), and the default bench line itself.
#   WLS="c5 c4 c2 c1 c3" tools/profile_round.sh <tag>
set -u
T=${1:-r02}
mkdir -p gpurun_out/profiles
B="python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e --no-unfused --no-gate --no-sub"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/launches_${T}.csv python bench.py --steps 5 --warmup 3 --no-cpu --no-sub > /dev/null 2>&1
ITEMS=""
for w in ${WLS:-c5 c4 c2 c1 c3}; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"fk_walk|fk_direct|fk_stream" -c 1 \
    -o gpurun_out/prof_${T}_$w $B --workload $w --steps 1 > gpurun_out/prof_${T}_$w.log 2>&1
  case $w in c3) K="C3[N=64]";; *) K=$(echo $w | tr a-z A-Z);; esac
  ITEMS="$ITEMS $K=gpurun_out/prof_${T}_$w.ncu-rep"
done
PROFILES_DIR=gpurun_out/profiles python tools/make_profiles.py $T $ITEMS --launches gpurun_out/launches_${T}.csv
[ "${KEEP:-0}" = 1 ] || rm -f gpurun_out/prof_${T}_*.ncu-rep
ls -la gpurun_out/profiles | tail -12
