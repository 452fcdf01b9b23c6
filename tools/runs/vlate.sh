# vertical path after the row's arrive (ASD_VLATE): parity with the variant, then A/B
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm --format=csv,noheader
ASD_LIB=$PWD/paper_2201_11924_b200/lib/variants/vlate.so timeout 600 python -m pytest tests/test_parity_gpu.py tests/test_batch_gpu.py -m gpu -q -x > gpurun_out/t_vlate.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/t_vlate.log
bash tools/ab.sh 2 base vlate
for v in base vlate base vlate; do
  echo "== bench $v"; ASD_LIB=$PWD/paper_2201_11924_b200/lib/variants/$v.so timeout 300 python bench.py --steps 5 --no-cpu-baseline --no-gate --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['clocks'])"
done
