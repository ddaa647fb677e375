#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
O=gpurun_out/exp2.txt; : > $O
for pass in 1 2; do
for c in 4 3 2; do
for lib in paper_1602_04386_b200/libfiedler.so build_variants/*.so; do
  echo "== pass $pass cfg $c $lib" >> $O
  FIEDLER_LIB=$PWD/$lib timeout 300 python tools/step_dist.py $c 20 >> $O 2>&1
done; done; done
