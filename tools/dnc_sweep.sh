#!/bin/bash
# superfast-vs-Schur-Levinson and block-size sweep for the large configs (one GPU)
cd "$(dirname "$0")/.."
run() { # cfg batch nt dncmin
  echo "== cfg$1 batch=$2 NT=$3 DNC_MIN=$4"
  SLSE_SOLVER_NT=$3 SLSE_DNC_MIN=$4 timeout ${5:-300} python tools/profile_step.py --config $1 --batch $2 --solves 2 --grids 0 2>&1 | grep -E "solve ms|k_hat|rror" | head -3
}
run 3 1024 256 1024
run 3 1024 128 1024
run 3 1024 512 1024
run 4 256 256 1024
run 4 256 512 1024
run 4 256 1024 1024
run 5 64 1024 1024 900
run 5 64 512 1024 900
