# config E (--job 4096), SGBM engine choice, D=256 ring depth, ncu of config-D directions
timeout 600 python bench.py --job 4096 --steps 3 --no-cpu-baseline --no-gate > gpurun_out/r01d_bench_jobE.json 2>gpurun_out/jobE.err; echo "jobE rc=$?"; cut -c1-300 gpurun_out/r01d_bench_jobE.json; tail -2 gpurun_out/jobE.err
for e in 1 3; do timeout 300 python bench.py --block 3 --engine $e --steps 5 --no-cpu-baseline --no-gate --no-e2e 2>/dev/null | cut -c1-120; done
for e in 1 3; do timeout 300 python bench.py --table2 128 --block 3 --engine $e --steps 5 2>/dev/null | cut -c1-150; done
for v in base d8p1 d8p3 d8p4; do echo "== $v"; ASD_LIB=$PWD/paper_2201_11924_b200/lib/variants/$v.so timeout 120 python tools/stage_times.py --engine 1 --reps 3 --config D --frames 8 --max-batch 8 2>&1 | grep -E "^  (dir|wta) |frames/s"; done
timeout 600 ncu --set full --import-source on --clock-control none -k regex:sgm_dir_kernel -s 9 -c 3 -o gpurun_out/r01d_d1_D python tools/stage_times.py --engine 1 --reps 1 --config D --frames 8 --max-batch 8 > gpurun_out/ncu_D.log 2>&1; echo "ncu D rc=$?"
