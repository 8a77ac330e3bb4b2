#!/bin/bash
# One ncu --set full capture of fbx_pipeline with the plan source (under gpurun):
#   TAG=<name> bash scripts/ncu_full.sh [bench args]
T=${TAG:-full}
mkdir -p gpurun_out
FBX_DUMP_SOURCE=gpurun_out/${T}.cu timeout 600 ncu --set full --clock-control none --import-source on -k regex:fbx_pipeline -s 3 -c 1 -o gpurun_out/${T} python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline "$@" > gpurun_out/${T}.log 2>&1
tail -c 300 gpurun_out/${T}.log
