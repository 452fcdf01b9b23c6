# D1 direction kernel: parity (D1 tests), A/B of variants, then the default bench line (with the D1 HBM gate)
timeout 900 python -m pytest tests -m gpu -q -x -k "D1 or fuzz or sgbm or r2 or batch" > gpurun_out/t_d1.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/t_d1.log
for cfgopt in "--config C --frames 32 --max-batch 32" "--config T96 --frames 32 --max-batch 32" "--config D --frames 8 --max-batch 8"; do
  echo "#### $cfgopt"
  for v in base minb8 pf2 l2x16 pf6; do
    echo "== $v"; ASD_LIB=$PWD/paper_2201_11924_b200/lib/variants/$v.so timeout 120 python tools/stage_times.py --engine 1 --reps 3 $cfgopt 2>&1 | grep -E "^  (dir) |frames/s"
  done
done
timeout 600 python bench.py > gpurun_out/bench_gate.json 2> gpurun_out/bench_gate.err; echo "bench rc=$?"; cat gpurun_out/bench_gate.json | cut -c1-3000
