# after the D = 256 census-load change: full GPU suite, smoke, headline bench, config D, Table II D=256
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/t_gpu_all.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/t_gpu_all.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke.log
timeout 600 python bench.py > gpurun_out/r01e_bench.json 2> gpurun_out/b.err; echo "bench rc=$?"; cut -c1-300 gpurun_out/r01e_bench.json
timeout 300 python bench.py --config D --frames 16 --steps 5 --no-cpu-baseline > gpurun_out/r01e_bench_configD.json 2>gpurun_out/cd.err; echo "configD rc=$?"; cut -c1-300 gpurun_out/r01e_bench_configD.json
rm -f gpurun_out/r01e_table2.jsonl
for D in 256; do timeout 300 python bench.py --table2 $D --steps 5 >> gpurun_out/r01e_table2.jsonl 2>>gpurun_out/t2.err; timeout 300 python bench.py --table2 $D --block 3 --steps 5 >> gpurun_out/r01e_table2.jsonl 2>>gpurun_out/t2.err; done
cut -c1-200 gpurun_out/r01e_table2.jsonl
