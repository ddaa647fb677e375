#!/bin/bash
# quick GPU round: parity subset, config-4 bench, setup phase times, timeline
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_dist_gpu.py -x -q -p no:cacheprovider > gpurun_out/dev_parity.log 2>&1; echo rc=$? >> gpurun_out/dev_parity.log
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/dev_bench4.log 2>&1
for c in ${PHASE_CFGS:-4 3}; do timeout 300 python tools/phase_times.py $c > gpurun_out/dev_phases_c$c.txt 2>&1; done
timeout 300 python tools/timeline_dump.py 4 > /dev/null 2>&1
