#!/bin/bash
# step-time distributions of every build_variants/*.so against the default library
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
O=gpurun_out/sweep_fracs.txt; : > $O
for c in ${CFGS:-4 3}; do
for lib in paper_1602_04386_b200/libfiedler.so build_variants/*.so; do
  echo "== cfg $c $lib" >> $O
  FIEDLER_LIB=$PWD/$lib timeout 300 python tools/step_dist.py $c ${REPS:-14} >> $O 2>&1
done; done
