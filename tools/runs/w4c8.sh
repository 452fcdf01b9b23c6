# WTA window rows of D + 4 u16 filled with 8-byte cp.async (half the fill instructions, 2-way bank conflicts on the diagonal) vs base
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm --format=csv,noheader
ASD_LIB=$PWD/paper_2201_11924_b200/lib/variants/w4c8.so timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/t_w4c8.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/t_w4c8.log
bash tools/ab.sh 2 base w4c8
for v in base w4c8 base w4c8; do
  echo "== bench $v"; ASD_LIB=$PWD/paper_2201_11924_b200/lib/variants/$v.so timeout 300 python bench.py --steps 5 --no-cpu-baseline --no-gate --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['clocks'])"
done
