#!/bin/bash
# per-level row-pass times of the default library and every build_variants/*.so (config CFG)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for lib in paper_1602_04386_b200/libfiedler.so build_variants/*.so; do
  echo "== $lib"
  FIEDLER_LIB=$PWD/$lib timeout 300 python tools/profile_levels.py ${CFG:-4} 10 2>&1 | head -${NL:-6}
done
