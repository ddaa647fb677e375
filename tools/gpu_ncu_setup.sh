#!/bin/bash
# ncu --set full of selected setup kernels of one create() on config CFG.  KRE=<kernel regex>
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
CFG=${CFG:-4}
KRE=${KRE:-"k_heavy_init|k_color_round|k_permute_rows|k_rs_scatter|k_repoint"}
timeout 600 python tools/profile_step.py $CFG 1 > gpurun_out/step_plain.log 2>&1 && \
timeout 1500 ncu --set full --clock-control none --import-source on -k "regex:$KRE" -c ${NK:-6} \
   -o gpurun_out/prof_setup -f python tools/profile_step.py $CFG 1 > gpurun_out/ncu_setup.log 2>&1
echo "ncu exit $?" >> gpurun_out/ncu_setup.log
tail -n 3 gpurun_out/ncu_setup.log
