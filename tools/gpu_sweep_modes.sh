#!/bin/bash
# create/solve host times of every build_variants/*.so, sweeps vs work lists
cd "$(dirname "$0")/.."
CFG=${CFG:-4}
for lib in build_variants/*.so; do
  for mode in 0 1; do
    echo "== $lib lists=$mode"
    FIEDLER_COOP_LISTS=$mode FIEDLER_LIB=$PWD/$lib timeout 300 python tools/profile_step.py $CFG 4 2>&1 | grep "rep [123]"
  done
done
