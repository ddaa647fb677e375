#!/bin/bash
# quick loop: -m gpu parity tests (excluding full-size), level profiles, benches of configs
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
T=${TAG:-q}
if [ -z "$NOTEST" ]; then
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider ${PYSEL:---deselect tests/test_gpu_fullsize.py} > gpurun_out/${T}_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_pytest.log
fi
for c in ${LEVCFGS:-2}; do timeout 600 python tools/profile_levels.py $c 5 > gpurun_out/${T}_lev$c.txt 2>&1; done
for c in ${BENCHCFGS:-2 4}; do timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 1 >> gpurun_out/${T}_bench.jsonl 2>> gpurun_out/${T}_bench.err; done
