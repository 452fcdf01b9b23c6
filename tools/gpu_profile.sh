#!/bin/bash
# ncu evidence for one tag (run under gpurun; one ncu tool per call):
#   tools/gpu_profile.sh TAG  ->  gpurun_out/TAG_launches.csv, TAG_full.ncu-rep
# The plain command runs first and must exit 0 (B200_PROFILING.md).
T=${1:-r02}
O=gpurun_out
CMD="python bench.py --steps 1 --warmup 3 --frames 22 --no-cpu-baseline --no-e2e --no-gate --no-parity"
python -c "import __graft_entry__ as g; g.build()" || exit 1
$CMD > $O/${T}_plain.json 2>&1 || exit 1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file $O/${T}_launches.csv $CMD > $O/${T}_ncu_l.log 2>&1; echo "launches rc=$?"
timeout 1500 ncu --set full --import-source on --clock-control none \
  -k regex:"census4|vsweep|hrow|wta2|lr_depth4" -s 12 -c 6 -o $O/${T}_full $CMD > $O/${T}_ncu_f.log 2>&1; echo "ncu full rc=$?"
