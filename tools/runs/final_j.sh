# round 1j: verify the WTA two-group fill commit (9a5b8b2) on a fresh box; new launch list + ncu full of the step kernels
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/r01j_gpu_tests.txt 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/r01j_gpu_tests.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')"
timeout 600 python bench.py > gpurun_out/r01j_bench.json 2> gpurun_out/b.err; echo "bench rc=$?"
cut -c1-600 gpurun_out/r01j_bench.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r01j_launches.csv python bench.py --steps 1 --warmup 3 --frames 22 --no-cpu-baseline --no-e2e --no-gate > gpurun_out/ncu_l.log 2>&1; echo "launches rc=$?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"census4|vsweep|hrow|wta2|lr_depth4" -s 12 -c 6 -o gpurun_out/r01j_full python bench.py --steps 1 --warmup 3 --frames 22 --no-cpu-baseline --no-e2e --no-gate > gpurun_out/ncu_f.log 2>&1; echo "ncu full rc=$?"
echo done
