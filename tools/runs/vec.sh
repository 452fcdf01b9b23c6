# D1 vectorised census loads: parity (D1 tests) + A/B vs the previous kernel
timeout 900 python -m pytest tests -m gpu -q -x -k "D1 or fuzz or sgbm or r2" > gpurun_out/t_vec.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/t_vec.log
for cfgopt in "--config C --frames 32 --max-batch 32" "--config D --frames 8 --max-batch 8" "--config T256 --frames 32 --max-batch 32" "--config T96 --frames 32 --max-batch 32" "--config T64 --frames 32 --max-batch 32"; do
  echo "#### $cfgopt"
  for v in base vec; do
    echo "== $v"; ASD_LIB=$PWD/paper_2201_11924_b200/lib/variants/$v.so timeout 120 python tools/stage_times.py --engine 1 --reps 3 $cfgopt 2>&1 | grep -E "^  dir |frames/s"
  done
done
