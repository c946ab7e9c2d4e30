#!/bin/bash
# ncu --set full with source correlation of one KD launch (default: alpha 0 of the second
# c3 forward of tools/prof_c3.py), exported as per-SASS-instruction CSV on the box.
#   bash tools/prof_kd_src.sh [regex] [tag] [skip]   (skip 1: alpha 0 of the second forward -- the only single-CTA launch of the NF = 8, Nt = 64 template at c3)
RE=${1:-'k_kd_tc<.int.8, .int.5, .bool.0, .int.64, .bool.0>'}
TAG=${2:-kd_a0}
python tools/prof_c3.py > gpurun_out/prof_plain.log 2>&1 || exit 1
ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:$RE" -s ${3:-1} -c 1 \
    -o "gpurun_out/$TAG" python tools/prof_c3.py > "gpurun_out/$TAG.log" 2>&1 || { echo "ncu failed"; exit 1; }
ncu -i "gpurun_out/$TAG.ncu-rep" --page source --csv --print-source sass > "gpurun_out/${TAG}_sass.csv" 2>&1
python tools/summarize_ncu_full.py "gpurun_out/$TAG.ncu-rep" > "gpurun_out/${TAG}_ncu.txt" 2>&1
rm -f "gpurun_out/$TAG.ncu-rep"
ls -la gpurun_out/${TAG}*
