#!/bin/bash
# ncu --set full of one launch of each named kernel (regex), from a short bench run.
# usage: TAG=r1e bash tools/ncu_kernels.sh 'k_ke' 'k_fft4_a<9, 8' ...
mkdir -p gpurun_out
i=0
for k in "$@"; do
  i=$((i+1))
  timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base ${KNB:-function} -k "regex:${k}" -s ${SKIP:-0} -c 1 \
    -o gpurun_out/${TAG:-r1e}_k${i} -f python bench.py --steps 1 --warmup 0 --no-cpu-baseline > gpurun_out/${TAG:-r1e}_k${i}.log 2>&1
  echo "kernel $i ($k): exit $?"
done
