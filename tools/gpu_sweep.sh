#!/bin/bash
# time level-0 row passes for every library variant under build_variants/
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
CFG=${CFG:-4}
for lib in build_variants/*.so; do
  echo "== $lib"
  FIEDLER_LIB=$PWD/$lib timeout 300 python tools/profile_levels.py $CFG 10 2>&1 | head -6
done > gpurun_out/sweep.log 2>&1
cat gpurun_out/sweep.log
