# D1 engine: parity + throughput (config C on D1, config D, Table II D=96/256)
set -x
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/t_d1.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/t_d1.log
timeout 300 python bench.py --engine 1 --steps 5 --no-cpu-baseline --no-e2e > gpurun_out/d1_C.json 2>gpurun_out/d1_C.err; cut -c1-1500 gpurun_out/d1_C.json
timeout 300 python bench.py --config D --frames 16 --steps 5 --no-cpu-baseline --no-e2e > gpurun_out/d1_D.json 2>gpurun_out/d1_D.err; cut -c1-1500 gpurun_out/d1_D.json
for D in 96 256; do timeout 300 python bench.py --table2 $D --steps 5 --no-cpu-baseline 2>>gpurun_out/t2.err | cut -c1-300; done
