set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/t_gpu.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/t_gpu.log
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
cat gpurun_out/bench.json
for D in 64 96 128 256; do timeout 300 python bench.py --table2 $D --steps 5 --no-cpu-baseline >> gpurun_out/table2.jsonl 2>>gpurun_out/table2.err; done
cut -c1-400 gpurun_out/table2.jsonl
