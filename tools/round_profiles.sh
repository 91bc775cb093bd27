# Round-end evidence on one GPU: bench line, launch list of the same bench
# command (cold, serialised), full ncu captures of the grid and solver kernels.
python bench.py > gpurun_out/bench.log 2>&1; echo bench_rc=$? >> gpurun_out/bench.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-cpu > gpurun_out/ncu_launches.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:grid_tma -c 1 -o gpurun_out/grid_full -f \
  python tools/grid_bench.py --reps 1 > gpurun_out/grid_ncu.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:solve_kernel -c 1 -o gpurun_out/solve_full -f \
  python tools/profile_step.py --config 2 --solves 1 --grids 0 > gpurun_out/solve_ncu.log 2>&1
