# WTA stage width (warps per CTA) at D = 128 in the pipelined step
timeout 600 python -m pytest tests -m gpu -q -x -k "C_full or batch" > gpurun_out/t_w.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/t_w.log
for r in 1 2; do
for v in ww8 ww4 ww6; do
  echo "== $v"; ASD_LIB=$PWD/paper_2201_11924_b200/lib/variants/$v.so timeout 120 python tools/stage_times.py --frames 128 --max-batch 22 --reps 3 2>&1 | grep -E "^  (row|wta|down) |frames/s"
done
done
