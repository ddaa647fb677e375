#!/bin/bash
# colouring-tail variants: phase times (FIEDLER_PHASE_TIMES) and step distributions of config 2
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for lib in paper_1602_04386_b200/libfiedler.so build_variants/*.so; do
  echo "== $lib"
  FIEDLER_LIB=$PWD/$lib timeout 300 python tools/phase_times.py 2 3 2>&1 | head -1
  FIEDLER_LIB=$PWD/$lib timeout 600 python tools/step_dist.py 2 15 2>&1 | tail -1
done
