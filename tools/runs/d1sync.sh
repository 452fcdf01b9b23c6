# new D1 fuzz cases; A/B of CTA width / vertical lock-step variants
timeout 900 python -m pytest tests/test_modes_fuzz_gpu.py -m gpu -q > gpurun_out/t_fuzz.log 2>&1; echo "fuzz rc=$?"; tail -2 gpurun_out/t_fuzz.log
for cfgopt in "--config C --frames 32 --max-batch 32" "--config D --frames 8 --max-batch 8"; do
  echo "#### $cfgopt"
  for v in base w8 w4s16 w8s16 w8s4; do
    echo "== $v"; ASD_LIB=$PWD/paper_2201_11924_b200/lib/variants/$v.so timeout 120 python tools/stage_times.py --engine 1 --reps 3 --timeline $cfgopt 2>&1 | grep -E "^  dir |frames/s" | tail -10
  done
done
