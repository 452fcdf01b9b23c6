# hrow: edge masks, whole-group specialisation, one-IMAD addressing -- parity + A/B
timeout 900 python -m pytest tests -m gpu -q -x -k "batch or C_full" > gpurun_out/t_hrow.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/t_hrow.log
for r in 1 2; do
for v in hbase hB hB4 hB3; do
  echo "== $v"; ASD_LIB=$PWD/paper_2201_11924_b200/lib/variants/$v.so timeout 120 python tools/stage_times.py --frames 128 --max-batch 22 --reps 3 2>&1 | grep -E "^  (row|wta|down) |frames/s"
done
done
