for kb in 12 14 16 20 27 40; do echo "region $kb KB" >> gpurun_out/occ47.log; SLSE_WARP_REGION_KB=$kb timeout 200 python tools/profile_step.py --solves 3 --grids 0 >> gpurun_out/occ47.log 2>&1; done
