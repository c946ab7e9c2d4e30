#!/bin/bash
# ncu --set full of one launch of every kernel class of the c3 forward (second forward of
# tools/prof_c3.py, 64 signals), one report per class: gpurun_out/r2_<name>.ncu-rep

run() {  # name regex skip
  ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:$2" -s "$3" -c 1 -o "gpurun_out/r2_$1" \
      python tools/prof_c3.py > "gpurun_out/r2_$1.log" 2>&1 || echo "ncu $1 failed" >> gpurun_out/r2_prof_errors.log
}
python tools/prof_c3.py > gpurun_out/prof_plain.log 2>&1
run ka 'k_fft4_a<.*ProbPad>' 1
run kb_a 'k_fft4_a<.int.9, .int.8, .*ProbFold>' 1
run kb_mid 'k_fft4_mid2<.int.9' 1
run kb_fin 'k_fft4_fin2<.int.9' 1
run kb_rows 'k_u1_fused<.int.12' 1
run kc_a 'k_fft4_a<.int.8, .int.8, .*ProbFold16>' 1
run kc_b 'k_fft4_b<.int.8, .int.8, .*ProbFold16>' 1
run kc_rows 'k_fft_rows<.int.12, .*ProbFold16>' 1
# summaries on the box (the reports themselves are large): profiles-ready text files
for f in gpurun_out/r2_*.ncu-rep; do
  n=$(basename "$f" .ncu-rep)
  python tools/summarize_ncu_full.py "$f" > "gpurun_out/${n}_ncu.txt" 2>&1
done
mkdir -p gpurun_out/keep
mv gpurun_out/r2_kb_a.ncu-rep gpurun_out/r2_kc_a.ncu-rep gpurun_out/keep/ 2>/dev/null || true
rm -f gpurun_out/r2_*.ncu-rep
