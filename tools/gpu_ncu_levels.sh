#!/bin/bash
# ncu --set full of the power-step pass on levels 1-3 and of one level-0 GS sweep + RQ (config CFG)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
CFG=${CFG:-4}
for L in ${LEVELS:-1 2 3}; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_tilepass -c 2 \
    -o gpurun_out/prof_pi_L${L} -f python tools/profile_kernel.py $CFG $L > gpurun_out/ncu_pi_L$L.log 2>&1
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_tilepass -s 2 -c 8 \
    -o gpurun_out/prof_gs_L0 -f python tools/profile_kernel.py $CFG 0 > gpurun_out/ncu_gs_L0.log 2>&1
