#!/bin/bash
# Round-end evidence (under gpurun): GPU tests, the default bench line, launch list
# (ncu gpu__time_duration), one ncu --set full capture of fbx_pipeline, traffic.
mkdir -p gpurun_out
python -m pytest tests -m gpu -q > gpurun_out/gputests.log 2>&1; tail -2 gpurun_out/gputests.log
python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -c 600 gpurun_out/bench.json
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
bash scripts/profile_kernel.sh ${PROF:-round_full}
