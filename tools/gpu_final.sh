#!/bin/bash
# round checkpoint: -m gpu suite, smoke, bench (driver default), other configs, sharded step on one GPU,
# ncu launch list of one config-4 step
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
TAG=${TAG:-ck}
timeout 2400 python -m pytest tests -m gpu -x -q -p no:cacheprovider --durations=8 > gpurun_out/${TAG}_pytest.log 2>&1; echo rc=$? >> gpurun_out/${TAG}_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1; echo rc=$? >> gpurun_out/${TAG}_smoke.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/${TAG}_bench4.jsonl 2> gpurun_out/${TAG}_bench4.err
for c in 1 2 3; do timeout 900 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline >> gpurun_out/${TAG}_bench_all.jsonl 2>> gpurun_out/${TAG}_bench_all.err; done
timeout 600 python bench.py --sharded --config 4 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/${TAG}_bench4_sharded.jsonl 2> gpurun_out/${TAG}_bench4_sharded.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/${TAG}_reference.jsonl 2> gpurun_out/${TAG}_reference.err
timeout 600 python tools/profile_step.py 4 1 > /dev/null 2>&1 && \
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 20000 --csv \
   --log-file gpurun_out/${TAG}_launches.csv python tools/profile_step.py 4 1 > gpurun_out/${TAG}_ncu_launch.log 2>&1
echo "launch list exit $?" >> gpurun_out/${TAG}_ncu_launch.log
