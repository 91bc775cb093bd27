#!/bin/bash
# superfast solver: block size x shared region x product-FFT flavour (one GPU)
cd "$(dirname "$0")/.."
run() { # cfg batch nt region_kb stockham timeout
  echo "== cfg$1 batch=$2 NT=$3 REGION=${4}KB DNC_STOCKHAM=$5"
  if [ "$5" = "1" ]; then export SLSE_DNC_STOCKHAM=1; else unset SLSE_DNC_STOCKHAM; fi
  SLSE_SOLVER_NT=$3 SLSE_DNC_MIN=1024 SLSE_REGION_KB=$4 timeout ${6:-300} python tools/profile_step.py --config $1 --batch $2 --solves 2 --grids 0 2>&1 | grep -E "solve ms|rror" | head -2
}
for nt in 32 64 128; do for reg in 16 64; do for sh in 0 1; do run 4 256 $nt $reg $sh; done; done; done
for nt in 32 64 128; do run 3 1024 $nt 16 0; run 3 1024 $nt 16 1; done
for nt in 32 64 128; do run 5 64 $nt 16 0 600; run 5 64 $nt 64 1 600; done
