#!/bin/bash
# build solver variants (launch-bounds min blocks for the one-warp solver) into build/variants/mbX/
cd "$(dirname "$0")/.."
for mb in "$@"; do
  sed -i "s/^#define SLSE_SOLVER_MINB32 .*/#define SLSE_SOLVER_MINB32 $mb/" paper_1705_06073_b200/csrc/slse_kernels.cuh
  python paper_1705_06073_b200/build.py --force > /dev/null
  mkdir -p build/variants/mb$mb && cp paper_1705_06073_b200/_lib/libsuperlse_b200.so build/variants/mb$mb/
done
