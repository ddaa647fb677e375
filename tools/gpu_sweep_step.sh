#!/bin/bash
# host-timed create/solve of config CFG for every library variant under build_variants/
cd "$(dirname "$0")/.."
CFG=${CFG:-4}
for lib in build_variants/*.so; do
  echo "== $lib"
  FIEDLER_LIB=$PWD/$lib timeout 300 python tools/profile_step.py $CFG 3 2>&1 | grep "rep [12]"
done
