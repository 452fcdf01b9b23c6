#!/bin/bash
# Cost of the segment-boundary exchange ("Frames wider than one
# cluster"): serialised launch durations (ncu) of the config-D sweeps on two
# segments against the same SEG instance on one segment (W = 960, forced with
# ASD_V2_FORCESEG in the ablation build).  Run under gpurun from the repo root:
#   ASD_VARIANT=abl ASD_NVCC_DEFS=-DASD_ABLATE python -m paper_2201_11924_b200.build
#   tools/seg_exp.sh   ->  gpurun_out/segx_{two,one}.csv
L=$PWD/paper_2201_11924_b200/lib/variants/abl.so
run() { tag=$1; w=$2; shift 2
  env ASD_LIB=$L "$@" timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:vsweep --csv \
    --log-file gpurun_out/segx_$tag.csv python tools/stage_times.py --config D --frames 6 --max-batch 6 --reps 1 \
    --width $w > gpurun_out/segx_$tag.log 2>&1
  echo "$tag rc=$?"; }
run two 1920 A=1
run one 960 ASD_V2_FORCESEG=1
