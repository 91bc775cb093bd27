#!/bin/bash
# cfg1 (one problem) solve time vs solver block size (knobs build).
cd "$(dirname "$0")/.."
export SLSE_LIB=build/variants/knobs/libsuperlse_b200.so
for nt in default 64 128 256 512; do
  if [ $nt = default ]; then unset SLSE_SOLVER_NT; else export SLSE_SOLVER_NT=$nt; fi
  echo "NT=$nt"; python tools/pair_ab.py 1 1 gpurun_out/nt_$nt.npz
done
python tools/pair_cmp.py gpurun_out/nt_default.npz gpurun_out/nt_128.npz
