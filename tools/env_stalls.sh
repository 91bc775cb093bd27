#!/bin/bash
# usage: tools/env_stalls.sh TAG "ENV=VAL ..." ["ENV=VAL ..."]  (on the GPU box)
# cfg2 solve time + warp-stall breakdown under each environment setting
tag=$1; shift
for envs in "$@"; do
  echo "== $envs" >> gpurun_out/env_$tag.log
  env $envs timeout 200 python tools/profile_step.py --solves 3 --grids 0 >> gpurun_out/env_$tag.log 2>&1
  env $envs timeout 300 ncu --section WarpStateStats --section InstructionStats --clock-control none -k regex:solve_kernel -c 1 --csv --page raw \
     python tools/profile_step.py --solves 1 --grids 0 2>/dev/null | python tools/stall_csv.py >> gpurun_out/env_$tag.log 2>&1
done
