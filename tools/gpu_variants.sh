#!/bin/bash
# create/solve host times of every build_variants/*.so (and the default lib)
cd "$(dirname "$0")/.."
for c in ${CFGS:-4 3}; do
for lib in build_variants/*.so paper_1602_04386_b200/libfiedler.so; do
  echo "== cfg $c $lib"
  FIEDLER_LIB=$PWD/$lib timeout 300 python tools/profile_step.py $c ${REPS:-5} 2>&1 | grep "^rep" | tail -n +2
done
done
