# Round-1d check: full GPU suite, smoke, Table II lines, config-D line
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/t_gpu_all.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/t_gpu_all.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke.log
rm -f gpurun_out/r01d_table2.jsonl
for D in 64 96 128 256; do timeout 300 python bench.py --table2 $D --steps 5 >> gpurun_out/r01d_table2.jsonl 2>>gpurun_out/t2.err; timeout 300 python bench.py --table2 $D --block 3 --steps 5 >> gpurun_out/r01d_table2.jsonl 2>>gpurun_out/t2.err; done
cut -c1-200 gpurun_out/r01d_table2.jsonl
timeout 300 python bench.py --config D --frames 16 --steps 5 --no-cpu-baseline --no-gate > gpurun_out/r01d_bench_configD.json 2>gpurun_out/cd.err; echo "configD rc=$?"; cut -c1-400 gpurun_out/r01d_bench_configD.json
timeout 300 python bench.py --engine 1 --steps 5 --no-cpu-baseline --no-gate > gpurun_out/r01d_bench_D1.json 2>gpurun_out/d1.err; echo "D1 rc=$?"; cut -c1-400 gpurun_out/r01d_bench_D1.json
