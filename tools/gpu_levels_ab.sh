#!/bin/bash
# per-level row-pass timings (CUDA events) of every build_variants/*.so and the default lib
cd "$(dirname "$0")/.."
for c in ${CFGS:-4}; do
for lib in build_variants/*.so paper_1602_04386_b200/libfiedler.so; do
  echo "== cfg $c $lib"
  FIEDLER_LIB=$PWD/$lib timeout 300 python tools/profile_levels.py $c ${REPS:-10} 2>&1 | grep -E "^L[0-9] |^sum"
done
done
