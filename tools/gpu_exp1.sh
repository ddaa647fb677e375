#!/bin/bash
# A/B: main-stream priority variant vs default; host time in pool calls (FIEDLER_ALLOC_STATS)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
O=gpurun_out/exp1.txt; : > $O
for c in 4 3 1; do
for lib in paper_1602_04386_b200/libfiedler.so build_variants/*.so; do
  echo "== cfg $c $lib" >> $O
  FIEDLER_LIB=$PWD/$lib timeout 300 python tools/step_dist.py $c 16 >> $O 2>&1
done; done
echo "== alloc stats cfg 4" >> $O
FIEDLER_ALLOC_STATS=1 timeout 300 python tools/profile_step.py 4 4 2>&1 | grep -v "^[0-9]" >> $O
FIEDLER_LIB=$PWD/build_variants/libfiedler_MAIN_PRIO1.so timeout 300 python tools/timeline_dump.py 4 create gpurun_out/timeline_create_c4_prio.json >> $O 2>&1
