#!/bin/bash
# segment-boundary exchange: parity subset, checked build (jitter) on the multi-cluster cases, config D line
timeout 900 python -m pytest tests/test_parity_gpu.py tests/test_modes_fuzz_gpu.py -x -q -k "two_segment or more_disparity or config_D or fuzz" 2>&1 | tail -1
ASD_LIB=$PWD/paper_2201_11924_b200/lib/variants/checked.so timeout 600 python tools/sanitize_cases.py --only seg128_d3,seg256_d3,C_d3,s128_d3 --repeat 5 2>&1 | tail -5
timeout 300 python bench.py --config D --steps 10 --warmup 3 --frames 32 --no-gate 2>/dev/null | cut -c1-400
