#!/bin/bash
# Round-2 grid (coefficient form) evidence: GPU grid tests, ncu --set full of
# grid_coef_kernel and grid_tma_kernel at the bench's roofline batch (43008),
# the default bench line and the bench's launch list.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "grid_eval" > gpurun_out/gc_tests.txt 2>&1
tail -2 gpurun_out/gc_tests.txt
timeout 300 ncu --set full --import-source on --clock-control none -k regex:grid_coef_kernel -s 2 -c 1 \
  -o gpurun_out/grid_coef -f python tools/grid_omega_bench.py --shapes 256:1024:43008 --reps 1 > gpurun_out/gc_ncu.log 2>&1
timeout 300 ncu --set full --import-source on --clock-control none -k regex:grid_tma_kernel -s 2 -c 1 \
  -o gpurun_out/grid_tma -f python tools/grid_bench.py --B 43008 --reps 1 > gpurun_out/gt_ncu.log 2>&1
timeout 1500 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
tail -c 600 gpurun_out/bench.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu --no-per-config > gpurun_out/ncu_bench.log 2>&1
echo done
