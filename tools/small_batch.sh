#!/bin/bash
# cfg2-shape solve time for small batches vs solver layout (knobs build):
# warp mode (16 one-warp solvers per CTA), classic one-warp CTAs, 128-thread CTAs.
cd "$(dirname "$0")/.."
export SLSE_LIB=build/variants/knobs/libsuperlse_b200.so
for B in ${BATCHES:-16 148 592 1184}; do
  echo "B=$B warps16"; python tools/pair_ab.py 2 $B /tmp/x.npz
  echo "B=$B classic32"; SLSE_NO_WARPS=1 python tools/pair_ab.py 2 $B /tmp/x.npz
  echo "B=$B nt128"; SLSE_SOLVER_NT=128 python tools/pair_ab.py 2 $B /tmp/x.npz
done
