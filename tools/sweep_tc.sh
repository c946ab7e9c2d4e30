#!/bin/bash
# KD tiling sweep: per-alpha KD ms for a few (NTMAX, SMAX) settings
for cfg in "256 8" "256 4" "128 8" "128 4" "64 8"; do
  set -- $cfg
  JTFS_TC_NTMAX=$1 JTFS_TC_SMAX=$2 timeout 300 python bench.py --steps 2 --warmup 3 --no-cpu-baseline 2>/dev/null | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print('NT<=$1 S<=$2', round(d['value'],1), 'KD', d['stages_ms']['KD_joint'], d['kd_ms_per_alpha'])"
done
