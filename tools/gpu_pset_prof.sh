#!/bin/bash
# ncu evidence of the partitioned-setup kernels (config 4, one rank owning every row):
# launch list of one partitioned setup + create_preset, and --set full of the
# first launch of the matching POINT, the JP colouring round and the per-row Galerkin
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 20000 --csv \
   --log-file gpurun_out/pset_launches.csv python tools/pset_phases.py 4 1048576 1 > gpurun_out/pset_ncu_launch.log 2>&1
echo "launch list exit $?" >> gpurun_out/pset_ncu_launch.log
for k in k_ps_point k_ps_colour k_ps_gal_small k_ps_q_join; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k -c 1 \
     -o gpurun_out/pset_$k -f python tools/pset_phases.py 4 1048576 1 > gpurun_out/pset_ncu_$k.log 2>&1
  echo "$k exit $?" >> gpurun_out/pset_ncu_$k.log
done
