#!/bin/bash
# Every reference bench experiment on the GPU (run under gpurun): CSVs in gpurun_out/fkbench/
set -u
mkdir -p gpurun_out/fkbench
for e in vf hf vf-hf ipo datasize datatype memory; do
  timeout 900 python -m paper_2508_07071_b200.fkbench $e --repeats ${REPEATS:-10} --csv gpurun_out/fkbench/$e.csv \
    2> gpurun_out/fkbench/$e.err
  echo "$e rc=$?"
done
