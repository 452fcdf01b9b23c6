# WIDE-key WTA ILP: fuzz parity, A/B (config D, Table II D=256, SGBM 3x3 config C), oracle single-core latency
timeout 900 python -m pytest tests/test_modes_fuzz_gpu.py tests/test_sgbm_gpu.py -m gpu -q > gpurun_out/t_wta.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/t_wta.log
for cfgopt in "--engine 1 --config D --frames 8 --max-batch 8" "--engine 1 --config T256 --frames 32 --max-batch 32" "--block 3 --frames 44 --max-batch 22" "--frames 88 --max-batch 22"; do
  echo "#### $cfgopt"
  for v in wtabase wtailp; do
    echo "== $v"; ASD_LIB=$PWD/paper_2201_11924_b200/lib/variants/$v.so timeout 120 python tools/stage_times.py --reps 3 $cfgopt 2>&1 | grep -E "^  (wta|dir|row) |frames/s"
  done
done
timeout 300 python tools/oracle_latency.py --out gpurun_out/r01d_oracle_latency.json; echo "oracle rc=$?"
