#!/bin/bash
# A/B the standalone cfg2 grid kernels in variant builds (build/variants/*),
# batch whose outputs exceed L2.  Usage: tools/grid_ab.sh name[:ENV=VAL] ...
cd "$(dirname "$0")/.."
B=${B:-10752}
for spec in "$@"; do
  v=${spec%%:*}; envs=""; [[ "$spec" == *:* ]] && envs=${spec#*:}
  echo "== $spec"; env $envs SLSE_LIB=build/variants/$v/libsuperlse_b200.so python tools/grid_bench.py --B $B --reps 30
done
