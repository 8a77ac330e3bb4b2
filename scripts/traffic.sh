#!/bin/bash
# DRAM traffic of one fbx_pipeline launch per DAG (ncu), -> gpurun_out/traffic_<dag>.csv
for d in ${DAGS:-sign_heavy default cross_heavy lookup_heavy fig4}; do
  ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
      -k regex:fbx_pipeline -s 3 -c 1 --csv --log-file gpurun_out/traffic_${d}.csv \
      python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --dag $d > /dev/null 2>&1
done
