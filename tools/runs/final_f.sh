# round-1f state: full GPU suite, smoke, bench (headline + gate), config D line, ncu launch list of the bench command, ncu full of hrow
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/t_gpu_all.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/t_gpu_all.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke.log
timeout 600 python bench.py > gpurun_out/r01f_bench.json 2> gpurun_out/b.err; echo "bench rc=$?"; cut -c1-300 gpurun_out/r01f_bench.json
timeout 300 python bench.py --config D --frames 16 --steps 5 --no-cpu-baseline > gpurun_out/r01f_bench_configD.json 2>gpurun_out/cd.err; echo "configD rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r01f_launches.csv python bench.py --steps 1 --warmup 3 --frames 22 --no-cpu-baseline --no-e2e --no-gate > gpurun_out/ncu_l.log 2>&1; echo "launches rc=$?"
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"hrow|wta2" -s 6 -c 2 -o gpurun_out/r01f_hrow python bench.py --steps 1 --warmup 3 --frames 22 --no-cpu-baseline --no-e2e --no-gate > gpurun_out/ncu_h.log 2>&1; echo "ncu hrow rc=$?"
