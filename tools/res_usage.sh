#!/bin/bash
# Registers / stack per kernel of lib/libfk_cuda.so whose mangled name matches $1.
cuobjdump -res-usage "$(dirname "$0")/../paper_2508_07071_b200/lib/libfk_cuda.so" 2>/dev/null |
  awk '/Function/ {f=$2} /REG:/ {print $1, $2, f}' | grep -E "${1:-.}" | sed 's/:$//'
