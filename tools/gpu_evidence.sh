#!/bin/bash
# round evidence: ncu launch list of one bench-style step, ncu --set full of the
# level-0 power step (dominant kernel; dram bytes -> profiles/traffic.json)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
CFG=${CFG:-4}
timeout 600 python tools/profile_step.py $CFG 2 > gpurun_out/ev_step_plain.log 2>&1 && \
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 20000 --csv \
   --log-file gpurun_out/ev_launches.csv python tools/profile_step.py $CFG 1 > gpurun_out/ev_ncu_launch.log 2>&1
echo "launch list exit $?" >> gpurun_out/ev_ncu_launch.log
timeout 600 python tools/profile_kernel.py $CFG 0 > gpurun_out/ev_kern_plain.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_tilepass -c 8 \
   -o gpurun_out/ev_prof_rowpass -f python tools/profile_kernel.py $CFG 0 > gpurun_out/ev_ncu_full.log 2>&1
echo "ncu full exit $?" >> gpurun_out/ev_ncu_full.log
