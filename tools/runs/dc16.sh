# sweep geometry: DC=32/T=4 (default) vs DC=16/T=8 in the current pipeline
for r in 1 2; do
  echo "== default"; timeout 120 python tools/stage_times.py --frames 128 --max-batch 22 --reps 3 2>&1 | grep -E "engine D3|^  (down|up|row|wta) |frames/s"
  echo "== dc16"; ASD_V2_DC16=1 timeout 120 python tools/stage_times.py --frames 128 --max-batch 22 --reps 3 2>&1 | grep -E "engine D3|^  (down|up|row|wta) |frames/s"
done
