#!/bin/bash
# One gpurun call: GPU tests, host-timed steps, ncu launch list of one step.  CFG=<config>
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
CFG=${CFG:-4}
if [ -z "$NOTEST" ]; then
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
fi
timeout 600 python tools/profile_step.py $CFG 3 > gpurun_out/step_plain.log 2>&1 && \
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 20000 --csv \
   --log-file gpurun_out/launches.csv python tools/profile_step.py $CFG 1 > gpurun_out/ncu_launch.log 2>&1
echo "launch list exit $?" >> gpurun_out/ncu_launch.log
tail -n 3 gpurun_out/pytest_gpu.log gpurun_out/ncu_launch.log; head -4 gpurun_out/step_plain.log
