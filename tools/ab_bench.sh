#!/bin/bash
# A/B of library variants on the headline bench line (no oracle, no e2e, no
# gate): tools/ab_bench.sh [rounds] lib1.so lib2.so ...  (paths relative to the repo)
R=${1:-2}; shift
for r in $(seq $R); do
  for v in "$@"; do
    printf "%-48s " "$v"
    ASD_LIB=$PWD/$v timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-gate --no-parity 2>/dev/null \
      | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],1), 'fps', {k: round(v/ (128*3) * 1000, 1) for k, v in d['stage_ms'].items()}, 'us/frame(prof)')"
  done
done
