#!/bin/bash
# ncu --set full of the level-0 setup kernels of config CFG (one create + solve)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
CFG=${CFG:-4}
TAG=${TAG:-setup}
timeout 300 python tools/profile_step.py $CFG 1 > gpurun_out/ncu_${TAG}_plain.log 2>&1 || exit 1
timeout 1500 ncu --set full --clock-control none --import-source on \
  -k regex:"${KREGEX:-k_match_coop|k_color_coop|k_gal_direct_batch|k_permute_rows|k_gal_write}" -c ${COUNT:-5} \
  -o gpurun_out/prof_${TAG} -f python tools/profile_step.py $CFG 1 > gpurun_out/ncu_${TAG}.log 2>&1
echo "ncu exit $?" >> gpurun_out/ncu_${TAG}.log
