# D3 A/B: sweep ring depths (pipelined wall frames/s at config C, 128 frames, max_batch 22)
for r in 1 2; do
for v in d3base ns6 ns8 ku5 ev1; do
  echo "== $v"; ASD_LIB=$PWD/paper_2201_11924_b200/lib/variants/$v.so timeout 120 python tools/stage_times.py --frames 128 --max-batch 22 --reps 3 2>&1 | grep -E "^  (down|up|row|wta|census) |frames/s"
done
done
