#!/bin/bash
# ncu --set full of grid_r3_kernel at the cfg3 / cfg4 / cfg5 roofline batches.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for spec in ${R3_SHAPES:-1024:4096:10752 4096:16384:2688}; do
  tag=$(echo $spec | tr ':' '_')
  timeout 300 ncu --set full --import-source on --clock-control none -k regex:grid_r3_kernel -s 2 -c 1 \
    -o gpurun_out/grid_r3_$tag -f python tools/grid_omega_bench.py --shapes $spec --reps 1 > gpurun_out/r3_ncu_$tag.log 2>&1
  tail -2 gpurun_out/r3_ncu_$tag.log
done
echo done
