#!/bin/bash
# Capture one ncu --set full profile of the fused kernel (run under gpurun, 1 GPU).
#   scripts/profile_kernel.sh <name> [bench args...]
name=${1:-prof}; shift
mkdir -p gpurun_out
FBX_DUMP_SOURCE=gpurun_out/${name}.cu ncu --set full --clock-control none --import-source on \
  -k regex:fbx_pipeline -s 3 -c 1 -o gpurun_out/${name} \
  python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline "$@" > gpurun_out/${name}.log 2>&1
tail -2 gpurun_out/${name}.log
python scripts/traffic.py gpurun_out/${name}.ncu-rep gpurun_out/${name}.log
