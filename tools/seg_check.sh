set -x
timeout 900 python -m pytest tests/test_parity_gpu.py -x -q -k "two_segment or more_disparity or config_D" 2>&1 | tail -3
timeout 300 python tools/sanitize_cases.py --only seg128_d3,seg256_d3,C_d3 --repeat 3 2>&1 | tail -4
for l in base.so ../libasd.so; do ASD_LIB=$PWD/paper_2201_11924_b200/lib/variants/$l timeout 300 python bench.py --config D --steps 5 --warmup 3 --frames 32 --no-cpu-baseline --no-e2e --no-gate --no-parity | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$l', round(d['value'],1), d['stage_ms'])"; done
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:vsweep --csv --log-file gpurun_out/segy_w1920.csv python tools/stage_times.py --config D --frames 6 --max-batch 6 --reps 1 > /dev/null 2>&1; echo ncu $?
