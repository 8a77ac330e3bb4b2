#!/bin/bash
# e2e throughput vs slice size (under gpurun)
for s in ${SLICES:-131072 262144 524288}; do
  python bench.py --steps ${STEPS:-10} --warmup 3 --no-cpu-baseline --e2e-slice-rows $s "$@" 2>/dev/null | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); e=d['e2e']; print('$s', round(e['value']/1e6,1), 'M rec/s stream;', round(e['single_step_value']/1e6,1), 'single;', e['digest'])"
done
