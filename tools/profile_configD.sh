T=r02d
O=gpurun_out
CMD="python bench.py --config D --steps 1 --warmup 3 --frames 6 --no-cpu-baseline --no-e2e --no-gate --no-parity"
$CMD > $O/${T}_plain.json 2>&1 || exit 1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file $O/${T}_launches.csv $CMD > $O/${T}_ncu_l.log 2>&1; echo "launches rc=$?"
timeout 1500 ncu --set full --import-source on --clock-control none \
  -k regex:"vsweep|hrow|wta2" -s 12 -c 4 -o $O/${T}_full $CMD > $O/${T}_ncu_f.log 2>&1; echo "ncu full rc=$?"
