#!/bin/bash
# One gpurun call: bench on the default workload, launch list of one step, ncu full of the rowpass.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
CFG=${CFG:-4}
timeout 900 python bench.py --config $CFG "$@" > gpurun_out/bench.log 2>&1; echo "bench exit $?" >> gpurun_out/bench.log
timeout 600 python tools/profile_step.py $CFG > gpurun_out/step_plain.log 2>&1 && \
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 20000 --csv \
   --log-file gpurun_out/launches.csv python tools/profile_step.py $CFG > gpurun_out/ncu_launch.log 2>&1
echo "launch list exit $?" >> gpurun_out/ncu_launch.log
timeout 600 python tools/profile_kernel.py $CFG 0 > gpurun_out/kern_plain.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_tilepass -c 8 \
   -o gpurun_out/prof_rowpass -f python tools/profile_kernel.py $CFG 0 > gpurun_out/ncu_full.log 2>&1
echo "ncu full exit $?" >> gpurun_out/ncu_full.log
tail -n 2 gpurun_out/bench.log gpurun_out/ncu_launch.log gpurun_out/ncu_full.log gpurun_out/kern_plain.log
