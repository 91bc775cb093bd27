#!/bin/bash
# A/B of grid_r3_kernel variants (build/variants/<name>, tools/capi_variant.sh)
cd "$(dirname "$0")/.."
for v in "$@"; do
  echo "== $v"
  SLSE_LIB=build/variants/$v/libsuperlse_b200.so python tools/grid_omega_bench.py --shapes ${R3_AB_SHAPES:-1024:4096:10752,4096:16384:2688,16384:65536:672} 2>&1 | grep -v '^ *$'
done
