# end-of-round state: bench lines, launch list, ncu full of the D3 kernels, Table II
timeout 600 python bench.py > gpurun_out/r01h_bench.json 2> gpurun_out/b.err; echo "bench rc=$?"; cut -c1-200 gpurun_out/r01h_bench.json
timeout 600 python bench.py --block 3 --steps 5 --no-cpu-baseline --no-gate > gpurun_out/r01h_bench_sgbm3.json 2>/dev/null; echo "sgbm rc=$?"
timeout 600 python bench.py --lr-mode 1 --steps 5 --no-cpu-baseline --no-gate > gpurun_out/r01h_bench_r2.json 2>/dev/null; echo "r2 rc=$?"
timeout 600 python bench.py --median 5 --steps 5 --no-cpu-baseline --no-gate > gpurun_out/r01h_bench_median5.json 2>/dev/null; echo "median rc=$?"
timeout 600 python bench.py --job 4096 --steps 3 --no-cpu-baseline --no-gate > gpurun_out/r01h_bench_jobE.json 2>/dev/null; echo "jobE rc=$?"
timeout 300 python bench.py --config D --frames 16 --steps 5 --no-cpu-baseline > gpurun_out/r01h_bench_configD.json 2>/dev/null; echo "configD rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r01h_launches.csv python bench.py --steps 1 --warmup 3 --frames 22 --no-cpu-baseline --no-e2e --no-gate > gpurun_out/ncu_l.log 2>&1; echo "launches rc=$?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"census4|vsweep|hrow|wta2|lr_depth4" -s 12 -c 6 -o gpurun_out/r01h_full python bench.py --steps 1 --warmup 3 --frames 22 --no-cpu-baseline --no-e2e --no-gate > gpurun_out/ncu_f.log 2>&1; echo "ncu full rc=$?"
rm -f gpurun_out/r01h_table2.jsonl
for D in 64 96 128 256; do timeout 300 python bench.py --table2 $D --steps 5 >> gpurun_out/r01h_table2.jsonl 2>/dev/null; timeout 300 python bench.py --table2 $D --block 3 --steps 5 >> gpurun_out/r01h_table2.jsonl 2>/dev/null; done
echo done
