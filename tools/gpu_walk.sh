#!/bin/bash
# fk_walk iteration: its tests, the bench-size parity tests, the C5/C4/C2 bench lines.
set -u
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_walk.py -x -q 2>&1 | tail -15
timeout 300 python -m pytest tests/test_gpu_bench_sizes.py -x -q -k "c5 or c4 or c2" 2>&1 | tail -5
bash tools/gpu_round.sh "${1:-c5 c4 c2}" "--co" 2>&1 | grep -v "^tests\|collected\|^$"
