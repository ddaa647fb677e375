#!/bin/bash
# GPU tests + a traced create/solve/destroy (FIEDLER_TRACE=1) + ncu full of the tile pass.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
CFG=${CFG:-4}
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
FIEDLER_TRACE=1 timeout 600 python tools/profile_step.py $CFG 3 > gpurun_out/trace.log 2>&1; echo "trace exit $?" >> gpurun_out/trace.log
if [ -z "$NONCU" ]; then
timeout 600 python tools/profile_kernel.py $CFG 0 > gpurun_out/kern_plain.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_tilepass -c 8 \
   -o gpurun_out/prof_rowpass -f python tools/profile_kernel.py $CFG 0 > gpurun_out/ncu_full.log 2>&1
echo "ncu full exit $?" >> gpurun_out/ncu_full.log
fi
tail -n 3 gpurun_out/pytest_gpu.log gpurun_out/ncu_full.log
