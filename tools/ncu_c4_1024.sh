#!/bin/bash
L=paper_2508_07071_b200/lib
cp $L/libfk_cuda.so /tmp/lib_main.so
for v in lib lib_6553ee3; do
  if [ "$v" = lib ]; then cp /tmp/lib_main.so $L/libfk_cuda.so; else cp paper_2508_07071_b200/$v/libfk_cuda.so $L/libfk_cuda.so; fi
  timeout 600 ncu --set full --clock-control none -k regex:fk_walk -c 1 -o gpurun_out/c4_1024_$v python bench.py --workload c4 --crops 1024 --steps 1 --warmup 3 --no-cpu --no-e2e --no-unfused --no-sub --no-gate > /dev/null 2>&1
done
cp /tmp/lib_main.so $L/libfk_cuda.so
