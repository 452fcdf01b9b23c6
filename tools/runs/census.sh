# byte-SIMD census: parity (every GPU test compares census bit-exact) + A/B
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/t_cen.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/t_cen.log
for r in 1 2; do
for v in wlbase wl; do
  echo "== $v"; ASD_LIB=$PWD/paper_2201_11924_b200/lib/variants/$v.so timeout 120 python tools/stage_times.py --frames 128 --max-batch 22 --reps 3 2>&1 | grep -E "^  (wta|row) |frames/s"
done
done
