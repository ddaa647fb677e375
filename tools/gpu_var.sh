#!/bin/bash
# create-time variance: P processes x 10 creates of config CFG (default 4)
cd "$(dirname "$0")/.."
CFG=${CFG:-4}
P=${P:-3}
for p in $(seq 1 $P); do
  timeout 300 python tools/profile_step.py $CFG 10 | grep "^rep" | awk '{print $6}' | tr '\n' ' '; echo
done
