#!/bin/bash
# Round-2 evidence for the L >= 4096 coefficient-form grid kernels (slse_grid3.cuh):
# ncu --set full of grid_r3_kernel (cfg3 shape) and grid_r3s_kernel (cfg4 / cfg5
# shapes) at the bench's roofline batches, then the default bench line and its launch list.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for spec in 1024:4096:10752:grid_r3c_kernel 4096:16384:2688:grid_r3s_kernel 16384:65536:672:grid_r3s_kernel; do
  IFS=: read n L B k <<< "$spec"
  timeout 300 ncu --set full --import-source on --clock-control none -k regex:$k -s 2 -c 1 \
    -o gpurun_out/${k}_n$n -f python tools/grid_omega_bench.py --shapes $n:$L:$B --reps 1 > gpurun_out/r3_ncu_n$n.log 2>&1
  tail -1 gpurun_out/r3_ncu_n$n.log
done
timeout 1500 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
tail -c 300 gpurun_out/bench.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu --no-per-config > gpurun_out/ncu_bench.log 2>&1
echo done
