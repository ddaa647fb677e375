#!/bin/bash
# create-time variance: 3 processes x 10 creates of config CFG (default 4)
cd "$(dirname "$0")/.."
CFG=${CFG:-4}
for p in 1 2 3; do
  timeout 300 python tools/profile_step.py $CFG 10 | grep "^rep" | awk '{print $6}' | tr '\n' ' '; echo
done
