#!/bin/bash
# sweep launch durations (ncu, serialised) at config C: with and without the per-row cluster barrier (timing only)
L=$PWD/paper_2201_11924_b200/lib/variants/abl.so
for ab in 0 2048 3072; do
  ASD_LIB=$L ASD_V2_ABLATE=$ab timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:vsweep --csv \
    --log-file gpurun_out/cb_$ab.csv python tools/stage_times.py --frames 11 --max-batch 11 --reps 1 > /dev/null 2>&1; echo "ab=$ab rc=$?"
done
