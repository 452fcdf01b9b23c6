#!/bin/bash
# A/B timing of kernel variants built into paper_2201_11924_b200/lib/variants/*.so:
#   tools/ab.sh [rounds] [variant ...]   (per-stage us/frame, config C, 11 frames)
R=${1:-2}; shift
V=${@:-$(ls paper_2201_11924_b200/lib/variants/ | sed 's/\.so$//')}
for r in $(seq $R); do
  for v in $V; do
    echo "== $v"
    ASD_LIB=$PWD/paper_2201_11924_b200/lib/variants/$v.so timeout 120 python tools/stage_times.py --frames 11 --max-batch 11 --reps 4 | grep -E "^  (down|up|row|wta|census) "
  done
done
