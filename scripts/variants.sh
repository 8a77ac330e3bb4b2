#!/bin/bash
# A/B code-generation knobs on the bench workload (under gpurun).
#   VARIANTS='FBX_MIN_BLOCKS=3;FBX_NVRTC_OPTS="-DA -DB"' scripts/variants.sh [bench args...]
IFS=";" read -ra VS <<< "${VARIANTS:-FBX_NONE=1}"
for rep in $(seq ${REPS:-1}); do
for v in "${VS[@]}"; do
  eval "env $v python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e $*" 2>&1 | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v $*', round(d['value']/1e9,3), 'Grec/s', d['roofline']['kernel_ms'], 'ms frac', d['roofline']['frac'], d['parity']['digest'])" 2>&1 | tail -1
done
done
