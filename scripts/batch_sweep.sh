# kernel time per chunk size / min-blocks bound (sign_heavy, 1M records)
for cfg in "256 4" "256 5" "128 8" "512 2" "${EXTRA:-}"; do
  set -- $cfg; [ -z "$1" ] && continue
  echo "bs=$1 mb=$2 $(FBX_MIN_BLOCKS=$2 python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu-baseline --batch-size $1 2>/tmp/err.txt | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["roofline"]["kernel_ms"], d["roofline"]["frac"])' 2>&1 | tail -1)"
done
