#!/bin/bash
# Standalone grid kernels at the cfg3/4/5 shapes (batches whose outputs
# exceed 2x L2) in variant builds (name[:ENV=VAL] ...).
cd "$(dirname "$0")/.."
for spec in "$@"; do
  v=${spec%%:*}; envs=""; [[ "$spec" == *:* ]] && envs=${spec#*:}
  for s in ${SHAPES:-"2688:1024:4096" "672:4096:16384" "168:16384:65536"}; do
    IFS=: read B N L <<< "$s"
    echo "== $spec B=$B N=$N L=$L"; env $envs SLSE_LIB=build/variants/$v/libsuperlse_b200.so python tools/grid_bench.py --B $B --N $N --L $L --reps 10
  done
done
