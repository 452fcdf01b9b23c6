#!/bin/bash
# One GPU-box verification pass (run under gpurun from the repo root):
#   tools/gpu_verify.sh TAG [steps]   ->  gpurun_out/TAG_*
# pytest -m gpu, smoke(), the default bench line (parity, e2e, cpu baseline,
# D1 gate), the side lines (config D, P2 = 40, SGBM 3x3, R2, Table II D = 96 /
# 256), the checked-build race/bounds run and the integer-pipe microbenchmark.
# Profiling (ncu) is a separate call: tools/gpu_profile.sh.
T=${1:-r02}; K=${2:-20}
O=gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/${T}_gpu.txt
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 1500 python -m pytest tests -m gpu -q -x > $O/${T}_gpu_tests.txt 2>&1; echo "pytest rc=$?"
tail -3 $O/${T}_gpu_tests.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/${T}_smoke.txt 2>&1; echo "smoke rc=$?"
timeout 900 python bench.py --steps $K --warmup 3 > $O/${T}_bench.json 2> $O/${T}_bench.err; echo "bench rc=$?"
cut -c1-300 $O/${T}_bench.json
for side in "configD:--config D --frames 32" "p2_40:--p2 40" "sgbm3:--block 3" "r2:--lr-mode 1"; do
  n=${side%%:*}; a=${side#*:}
  timeout 900 python bench.py --steps 10 --warmup 3 --no-gate $a > $O/${T}_bench_$n.json 2>> $O/${T}_bench.err; echo "bench $n rc=$?"
done
for d in 64 96 128 256; do timeout 600 python bench.py --table2 $d --steps 10 --warmup 3 --frames 64 >> $O/${T}_table2.jsonl 2>> $O/${T}_bench.err; done
timeout 900 tools/checked.sh 5 > $O/${T}_checked.txt 2>&1; echo "checked rc=$?"
tail -2 $O/${T}_checked.txt
mkdir -p build && nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o build/ubench tools/ubench.cu && ./build/ubench > $O/${T}_ubench.txt 2>&1
cat $O/${T}_ubench.txt
