#!/bin/bash
# A/B: persisting-L2 window for the colouring's byte state (FIEDLER_L2_PERSIST=1)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
O=gpurun_out/exp5.txt; : > $O
for pass in 1 2; do
for c in 4 3 1; do
for on in 0 1; do
  echo "== pass $pass cfg $c L2_PERSIST=$on" >> $O
  FIEDLER_L2_PERSIST=$on timeout 300 python tools/step_dist.py $c 16 >> $O 2>&1
done; done; done
FIEDLER_L2_PERSIST=1 timeout 300 python tools/phase_times.py 4 > gpurun_out/exp5_phases_on.txt 2>&1
FIEDLER_L2_PERSIST=0 timeout 300 python tools/phase_times.py 4 > gpurun_out/exp5_phases_off.txt 2>&1
