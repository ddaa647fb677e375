#!/bin/bash
# sharded step on one GPU: main-stream priority on / off
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
O=gpurun_out/exp6.txt; : > $O
for pass in 1 2; do
for lib in paper_1602_04386_b200/libfiedler.so build_variants/libfiedler_MAIN_PRIO0.so; do
  echo "== pass $pass $lib" >> $O
  FIEDLER_LIB=$PWD/$lib timeout 600 python bench.py --sharded --config 4 --steps 6 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys
l=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(l['ms_per_step'], l['replicas']['ms_per_step'])" >> $O 2>&1
done; done
