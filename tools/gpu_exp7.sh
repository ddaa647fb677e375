#!/bin/bash
# deferred layouts of the big levels: parity, then step-time sweep of the thresholds
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
O=gpurun_out/exp7.txt; : > $O
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_dist_gpu.py -m gpu -x -q -p no:cacheprovider > gpurun_out/exp7_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/exp7_pytest.log
tail -3 gpurun_out/exp7_pytest.log >> $O
for c in 4 3; do
for lib in paper_1602_04386_b200/libfiedler.so build_variants/*.so; do
  echo "== cfg $c $lib" >> $O
  FIEDLER_LIB=$PWD/$lib timeout 300 python tools/step_dist.py $c 14 >> $O 2>&1
done; done
for c in 1 2; do
for lib in paper_1602_04386_b200/libfiedler.so build_variants/libfiedler_DEFER_NNZ0.so; do
  echo "== cfg $c $lib" >> $O
  FIEDLER_LIB=$PWD/$lib timeout 300 python tools/step_dist.py $c 14 >> $O 2>&1
done; done
