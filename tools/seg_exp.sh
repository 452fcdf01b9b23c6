#!/bin/bash
timeout 900 python -m pytest tests/test_parity_gpu.py tests/test_modes_fuzz_gpu.py tests/test_batch_gpu.py -x -q 2>&1 | tail -2
tools/ab_line.sh "--config D --frames 32" 2 paper_2201_11924_b200/lib/variants/cur.so paper_2201_11924_b200/lib/variants/split.so
