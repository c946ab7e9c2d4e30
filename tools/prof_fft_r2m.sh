run() {
  ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:$2" -s "$3" -c 1 -o "gpurun_out/r2m_$1" \
      python tools/prof_c3.py > "gpurun_out/r2m_$1.log" 2>&1 || echo "ncu $1 failed"
  python tools/summarize_ncu_full.py "gpurun_out/r2m_$1.ncu-rep" > "gpurun_out/r2m_$1_ncu.txt" 2>&1
  rm -f "gpurun_out/r2m_$1.ncu-rep"
}
python tools/prof_c3.py > gpurun_out/prof_plain.log 2>&1
run kc_a 'k_fft4_a<.int.8, .int.8, .*ProbFold16>' 1
run kc_b 'k_fft4_b<.int.8, .int.8, .*ProbFold16>' 1
run kb_a 'k_fft4_a<.int.9, .int.8, .*ProbFold>' 1
for f in kc_a kc_b kb_a; do echo "== $f"; grep -E "gpu__time_duration|dram__bytes_read|dram__bytes_write|long_scoreboard" gpurun_out/r2m_${f}_ncu.txt; done
