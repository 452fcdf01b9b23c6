#!/bin/bash
# A/B of two library builds (cur, new) on the headline, R2, config D and Table II D = 128 lines (value only)
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -1
for r in 1 2; do for v in cur new; do for a in "" "--lr-mode 1" "--config D --frames 32" "--table2 128 --frames 64"; do
  printf "%-4s %-26s " $v "$a"
  ASD_LIB=$PWD/paper_2201_11924_b200/lib/variants/$v.so timeout 600 python bench.py $a --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-gate --no-parity 2>/dev/null | python -c "import json,sys; print(round(json.loads(sys.stdin.read())['value'],1))"
done; done; done
