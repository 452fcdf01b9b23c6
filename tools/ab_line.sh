#!/bin/bash
# A/B of library variants on any bench line: tools/ab_line.sh "bench args" rounds lib.so ...
A="$1"; R=${2:-2}; shift 2
for r in $(seq $R); do
  for v in "$@"; do
    printf "%-48s " "$v"
    ASD_LIB=$PWD/$v timeout 600 python bench.py $A --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-gate --no-parity 2>/dev/null \
      | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],1), 'fps', {k: round(v, 1) for k, v in d['stage_ms'].items()})"
  done
done
