#!/bin/bash
# ReduceDPP kernel times (ncu) for lib and each lib_<tag> given: tools/ab_reduce.sh u1 u4
set -u
L=paper_2508_07071_b200/lib
cp $L/libfk_cuda.so /tmp/libA.so
for t in A "$@"; do
  [ $t != A ] && cp paper_2508_07071_b200/lib_$t/libfk_cuda.so $L/libfk_cuda.so
  echo "== $t"
  ncu --metrics gpu__time_duration.sum --clock-control none -k regex:fk_reduce_plain --csv python tools/reduce_probe.py 2>/dev/null | python tools/ncu_times.py 13
  cp /tmp/libA.so $L/libfk_cuda.so
done
