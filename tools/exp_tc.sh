#!/bin/bash
for m in 0 2 4; do
  JTFS_TC_EXPMODE=$m timeout 300 python bench.py --steps 2 --warmup 3 --no-cpu-baseline 2>/dev/null | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print('expmode $m', round(d['value'],1), 'KD', d['stages_ms']['KD_joint'], d['kd_ms_per_alpha'])"
done
