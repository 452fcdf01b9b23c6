#!/bin/bash
# One GPU-box verification pass (run under gpurun from the repo root):
#   tools/gpu_verify.sh TAG [steps]   ->  gpurun_out/TAG_*.{txt,json,log}
# pytest -m gpu, smoke(), the checked-build race/bounds run, the default bench
# line, the integer-pipe microbenchmark.  Profiling (ncu) is a separate call.
T=${1:-r02}; K=${2:-20}
O=gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/${T}_gpu.txt
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 1200 python -m pytest tests -m gpu -q -x > $O/${T}_gpu_tests.txt 2>&1; echo "pytest rc=$?"
tail -3 $O/${T}_gpu_tests.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/${T}_smoke.txt 2>&1; echo "smoke rc=$?"
timeout 600 python bench.py --steps $K --warmup 3 > $O/${T}_bench.json 2> $O/${T}_bench.err; echo "bench rc=$?"
cut -c1-400 $O/${T}_bench.json
timeout 900 tools/checked.sh 5 > $O/${T}_checked.txt 2>&1; echo "checked rc=$?"
tail -2 $O/${T}_checked.txt
mkdir -p build && nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o build/ubench tools/ubench.cu && ./build/ubench > $O/${T}_ubench.txt 2>&1
cat $O/${T}_ubench.txt
