#!/bin/bash
# step-time distributions: every library x {deferred level 0, eager level 0}
cd "$(dirname "$0")/.."
for c in ${CFGS:-4}; do
for lib in paper_1602_04386_b200/libfiedler.so build_variants/*.so; do
  for e in 0 1; do
    echo "== $lib eager_l0=$e"
    FIEDLER_EAGER_L0=$e FIEDLER_LIB=$PWD/$lib timeout 600 python tools/step_dist.py $c ${REPS:-15} 2>&1 | tail -1
  done
done
done
