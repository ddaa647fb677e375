#!/bin/bash
# quick loop: GPU tests (optional) + level-0 kernel timings on config CFG
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
CFG=${CFG:-4}
if [ -z "$NOTEST" ]; then
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
tail -n 2 gpurun_out/pytest_gpu.log
fi
timeout 600 python tools/profile_kernel.py $CFG 0 10 > gpurun_out/kern_plain.log 2>&1; cat gpurun_out/kern_plain.log
FIEDLER_TRACE=1 timeout 600 python tools/profile_step.py $CFG 2 > gpurun_out/trace.log 2>&1; grep "rep\|setup_ms" gpurun_out/trace.log
