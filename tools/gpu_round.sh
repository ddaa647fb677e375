#!/bin/bash
# tests + quick timings + variant sweep
cd "$(dirname "$0")/.."
tools/gpu_quick.sh
tools/gpu_sweep.sh
