#!/bin/bash
# Round-2 evidence pass (under gpurun, 1 GPU): bench line per Appendix-B DAG (with the
# drop-in run_pipelined e2e), launch list, ncu --set full of fbx_pipeline for
# sign_heavy with its DRAM traffic recorded in profiles/traffic.json (plan-hashed).
mkdir -p gpurun_out
for d in ${DAGS:-sign_heavy cross_heavy lookup_heavy default fig4}; do
  timeout 600 python bench.py --dag $d --no-cpu-baseline 2>gpurun_out/r2_bench_$d.err | tail -1 > gpurun_out/r2_bench_$d.json
  python -c "import json;d=json.load(open('gpurun_out/r2_bench_$d.json'));r=d['roofline'];print('$d', d['value'], r['kernel_ms'], r['frac'], r['index_build_ms'], d['e2e']['value'], d['parity']['shards_checked'])"
done
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv \
  --log-file gpurun_out/r2_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
for d in ${PROF_DAGS:-sign_heavy}; do
  FBX_DUMP_SOURCE=gpurun_out/r2_full_$d.cu timeout 600 ncu --set full --clock-control none --import-source on \
    -k regex:fbx_pipeline -s 3 -c 1 -o gpurun_out/r2_full_$d python bench.py --dag $d --steps 1 --warmup 3 \
    --no-e2e --no-cpu-baseline > gpurun_out/r2_full_$d.log 2>&1
  python scripts/traffic.py gpurun_out/r2_full_$d.ncu-rep gpurun_out/r2_full_$d.log
done
# C5: 100 independent shards (default DAG), shards over 3 streams, run_pipelined per shard
timeout 1200 python bench.py --dag default --shards 100 --steps 3 --warmup 3 --no-cpu-baseline \
  2>gpurun_out/r2_bench_c5.err | tail -1 > gpurun_out/r2_bench_c5.json
python -c "import json;d=json.load(open('gpurun_out/r2_bench_c5.json'));print('C5', d['value'], d['ms_per_step'], d['e2e']['value'], d['parity']['shards_checked'])"
# the default bench line with its cpu baseline (the driver's own run)
timeout 900 python bench.py > gpurun_out/r2_bench_default_full.json 2>gpurun_out/r2_bench_default_full.err
python scripts/pcie_probe.py > gpurun_out/r2_pcie.txt 2>&1
