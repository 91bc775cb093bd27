#!/bin/bash
cd "$(dirname "$0")/.."
for mb in 12 16 24; do
  for reg in 12 16; do
    echo "== mb=$mb region=${reg}KB"
    SLSE_LIB=build/variants/mb$mb/libsuperlse_b200.so SLSE_WARP_REGION_KB=$reg timeout 300 python tools/profile_step.py --config 2 --batch 4096 --solves 3 --grids 0 2>&1 | grep -E "solve ms|Error" | head -2
  done
done
