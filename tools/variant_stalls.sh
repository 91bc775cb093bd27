#!/bin/bash
# usage: tools/variant_stalls.sh OUT_TAG lib1 lib2 ...  (on the GPU box)
# times a cfg2 solve with each library and records the warp-stall breakdown
tag=$1; shift
for lib in "$@"; do
  echo "== $lib" >> gpurun_out/var_$tag.log
  SLSE_LIB=$lib timeout 200 python tools/profile_step.py --solves 3 --grids 0 >> gpurun_out/var_$tag.log 2>&1
  SLSE_LIB=$lib timeout 300 ncu --section WarpStateStats --section InstructionStats --clock-control none -k regex:solve_kernel -c 1 --csv --page raw \
     python tools/profile_step.py --solves 1 --grids 0 2>/dev/null | python tools/stall_csv.py >> gpurun_out/var_$tag.log 2>&1
done
