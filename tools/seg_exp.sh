#!/bin/bash
# config D pipeline with forced cluster sizes (ablation build)
for cs in 0 16 8 10 12; do echo "cs=$cs"; ASD_V2_CS=$cs tools/ab_line.sh "--config D --frames 32" 1 paper_2201_11924_b200/lib/variants/abl.so; done
