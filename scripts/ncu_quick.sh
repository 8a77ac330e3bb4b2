#!/bin/bash
# Key metrics of fbx_pipeline for env variants: VARIANTS="A=1;A=0" scripts/ncu_quick.sh [bench args]
IFS=";" read -ra VS <<< "${VARIANTS:-FBX_NONE=1}"
M=gpu__time_duration.sum,smsp__inst_executed.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,smsp__thread_inst_executed_per_inst_executed.ratio,l1tex__t_bytes_pipe_lsu_mem_local_op_ld.sum,lts__t_bytes.sum,sm__warps_active.avg.pct_of_peak_sustained_active,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio,smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio
mkdir -p gpurun_out
i=0
for v in "${VS[@]}"; do
  i=$((i+1))
  eval "env $v ncu --metrics $M --clock-control none -k regex:fbx_pipeline -s 3 -c 1 --csv --log-file gpurun_out/q$i.csv python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline $*" > /dev/null 2>&1
  python -c "
import csv
rows=[r for r in csv.reader(open('gpurun_out/q$i.csv')) if len(r)>10]
h=rows[0]; mi=h.index('Metric Name'); vi=h.index('Metric Value')
print('$v', ' | '.join(r[mi].split('.')[0][-30:] + '=' + r[vi] for r in rows[1:]))"
done
