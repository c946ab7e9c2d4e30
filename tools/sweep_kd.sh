#!/bin/bash
# KD tile-width sweep (per-alpha KD ms): Nt <= NTMAX; TMEM buffers per epilogue set = 256 / Nt
for nt in 256 128 64; do
  JTFS_TC_NTMAX=$nt timeout 300 python bench.py --steps 2 --warmup 3 --no-cpu-baseline 2>/dev/null | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print('NTMAX=$nt', round(d['value'],1), 'KD', d['stages_ms']['KD_joint'], d['kd_ms_per_alpha'])"
done
