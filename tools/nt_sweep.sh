#!/bin/bash
# Solver block-size sweep (one GPU): prints solve ms per config / NT.
cd "$(dirname "$0")/.."
for cfg_nt in "2:32" "2:64" "2:128" "2:256" "3:32" "3:64" "3:128" "3:256" "3:512" "4:256" "4:512" "4:1024"; do
  cfg=${cfg_nt%%:*}; nt=${cfg_nt##*:}
  case $cfg in 2) b=4096;; 3) b=1024;; 4) b=256;; esac
  echo "== cfg$cfg NT=$nt batch=$b"
  SLSE_SOLVER_NT=$nt timeout 300 python tools/profile_step.py --config $cfg --batch $b --solves 2 --grids 0 2>&1 | grep -E "solve ms|k_hat|Error|error" | head -3
done
echo "== cfg5 NT=1024 batch=8"
SLSE_SOLVER_NT=1024 timeout 600 python tools/profile_step.py --config 5 --batch 8 --solves 1 --grids 0 2>&1 | tail -3
