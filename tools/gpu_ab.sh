#!/bin/bash
# A/B host timing of library variants: LIBS="a.so b.so" CFGS="4" REPS=4 bash tools/gpu_ab.sh
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
CFGS=${CFGS:-4}
REPS=${REPS:-4}
for cfg in $CFGS; do
  for round in 1 2; do
    for lib in $LIBS; do
      echo "== cfg $cfg lib $lib round $round"
      FIEDLER_LIB=$lib timeout 600 python tools/profile_step.py $cfg $REPS 2>&1 | grep "^rep" | tail -n +2
    done
  done
done
