#!/bin/bash
# step-time distributions of the default library and every build_variants/*.so
cd "$(dirname "$0")/.."
for c in ${CFGS:-4}; do
for lib in paper_1602_04386_b200/libfiedler.so build_variants/*.so; do
  echo "== $lib"
  FIEDLER_LIB=$PWD/$lib timeout 600 python tools/step_dist.py $c ${REPS:-30} 2>&1 | tail -1
done
done
