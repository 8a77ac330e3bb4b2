#!/bin/bash
# Round-2 profiling pass (under gpurun, 1 GPU): bench line (kernel + index build),
# launch list, ncu --set full of fbx_pipeline and of the basic index build, phase timers.
#   TAG=<name> bash scripts/gpu_profile_r2.sh [bench args]
T=${TAG:-p}
mkdir -p gpurun_out
timeout 300 python bench.py --no-e2e --no-cpu-baseline "$@" > gpurun_out/${T}_bench.log 2>&1; tail -c 1500 gpurun_out/${T}_bench.log | grep -o '"kernel_ms[^}]*'
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/${T}_launches.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline "$@" > /dev/null 2>&1
FBX_DUMP_SOURCE=gpurun_out/${T}_full.cu timeout 600 ncu --set full --clock-control none --import-source on -k regex:fbx_pipeline -s 3 -c 1 -o gpurun_out/${T}_full python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline "$@" > gpurun_out/${T}_full.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:fbx_side_prep_1 -s 2 -c 1 -o gpurun_out/${T}_prep python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline "$@" > gpurun_out/${T}_prep.log 2>&1
FBX_PHASE_TIMERS=1 timeout 300 python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline "$@" 2>&1 | grep FBX_PHASE | tail -10 > gpurun_out/${T}_phases.txt
cat gpurun_out/${T}_phases.txt
