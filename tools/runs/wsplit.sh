# WTA window fill in two commit groups (ASD_WTA_SPLIT): parity with the variant, then A/B
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm --format=csv,noheader
ASD_LIB=$PWD/paper_2201_11924_b200/lib/variants/split.so timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/t_split.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/t_split.log
bash tools/ab.sh 2 base split
for v in base split base split; do
  echo "== bench $v"; ASD_LIB=$PWD/paper_2201_11924_b200/lib/variants/$v.so timeout 300 python bench.py --steps 5 --no-cpu-baseline --no-gate --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['clocks'])"
done
