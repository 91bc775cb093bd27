#!/bin/bash
# cfg2 solve time vs batch size (tail effect), warp mode and free mode
for b in 2368 4096 4736 8192; do
  echo "B=$b warps" >> gpurun_out/bsweep_$1.log
  timeout 200 python tools/profile_step.py --batch $b --solves 3 --grids 0 2>&1 | grep solve >> gpurun_out/bsweep_$1.log
  echo "B=$b free" >> gpurun_out/bsweep_$1.log
  SLSE_NO_WARPS=1 timeout 200 python tools/profile_step.py --batch $b --solves 3 --grids 0 2>&1 | grep solve >> gpurun_out/bsweep_$1.log
done
