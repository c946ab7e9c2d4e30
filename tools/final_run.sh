set -x
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/f_smoke.log 2>&1; echo smoke=$?
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/f_gput.log 2>&1; echo gput=$?; tail -3 gpurun_out/f_gput.log
timeout 600 python bench.py > gpurun_out/f_bench_c3.json 2> gpurun_out/f_bench_c3.err; echo bench=$?
for w in c2 c4 scat1d resynth; do timeout 300 python bench.py --workload $w --no-cpu-baseline > gpurun_out/f_bench_$w.json 2> gpurun_out/f_bench_$w.err; echo $w=$?; done
timeout 300 python bench.py --impl reference --steps 1 --warmup 0 > gpurun_out/f_bench_ref.json 2> gpurun_out/f_bench_ref.err; echo ref=$?
