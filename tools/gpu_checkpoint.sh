#!/bin/bash
# full round checkpoint: -m gpu suite, smoke, bench (driver's default), other configs, phase times
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
TAG=${TAG:-ck}
timeout 2400 python -m pytest tests -m gpu -x -q -p no:cacheprovider --durations=8 > gpurun_out/${TAG}_pytest.log 2>&1; echo rc=$? >> gpurun_out/${TAG}_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1; echo rc=$? >> gpurun_out/${TAG}_smoke.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/${TAG}_bench4.jsonl 2> gpurun_out/${TAG}_bench4.err
for c in 1 2 3; do timeout 900 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline >> gpurun_out/${TAG}_bench_all.jsonl 2>> gpurun_out/${TAG}_bench_all.err; done
for c in 4 3; do timeout 300 python tools/phase_times.py $c > gpurun_out/${TAG}_phases_c$c.txt 2>&1; done
