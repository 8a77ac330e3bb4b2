#!/bin/bash
# Bench line per SURVEY config (C2 sign_heavy, C3 cross_heavy, C4 lookup_heavy, default, fig4, C5 shards)
mkdir -p gpurun_out
python scripts/pcie_probe.py > gpurun_out/pcie.txt 2>&1
for d in ${DAGS:-sign_heavy cross_heavy lookup_heavy default fig4}; do
  python bench.py --dag $d --no-cpu-baseline ${EXTRA} 2>gpurun_out/bench_$d.err | tail -1 > gpurun_out/bench_$d.json
done
if [ -z "$NO_C5" ]; then
  python bench.py --dag default --shards ${SHARDS:-8} --no-cpu-baseline --no-e2e 2>gpurun_out/bench_c5.err | tail -1 > gpurun_out/bench_c5.json
fi
