#!/bin/bash
cd "$(dirname "$0")/.."
for c in 4 3 2; do
for lib in build_variants/*.so; do
  echo "== cfg $c $lib"
  FIEDLER_COOP_LISTS=1 FIEDLER_LIB=$PWD/$lib timeout 300 python tools/profile_step.py $c 4 2>&1 | grep "rep [123]"
done
done
FIEDLER_COOP_LISTS=1 timeout 300 python tools/phase_times.py 4 > gpurun_out/phases_c4_lists.txt 2>&1
FIEDLER_COOP_LISTS=0 timeout 300 python tools/phase_times.py 4 > gpurun_out/phases_c4_sweeps.txt 2>&1
FIEDLER_SERIAL_COLOUR=1 FIEDLER_COOP_LISTS=1 timeout 300 python tools/phase_times.py 4 > gpurun_out/phases_c4_lists_serial.txt 2>&1
FIEDLER_SERIAL_COLOUR=1 FIEDLER_COOP_LISTS=0 timeout 300 python tools/phase_times.py 4 > gpurun_out/phases_c4_sweeps_serial.txt 2>&1
FIEDLER_COOP_LISTS=1 timeout 300 python tools/phase_times.py 3 > gpurun_out/phases_c3_lists.txt 2>&1
FIEDLER_COOP_LISTS=1 timeout 300 python tools/phase_times.py 2 > gpurun_out/phases_c2_lists.txt 2>&1
