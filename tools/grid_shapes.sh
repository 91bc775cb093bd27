#!/bin/bash
# Standalone grid kernels at the cfg3/4/5 shapes (batches whose outputs
# exceed 2x L2) in variant builds; SLSE_GRID_OLD=1 selects the previous dispatch.
cd "$(dirname "$0")/.."
for spec in "$@"; do
  v=${spec%%:*}; envs=""; [[ "$spec" == *:* ]] && envs=${spec#*:}
  for s in "2688 1024 4096" "672 4096 16384" "168 16384 65536"; do
    set -- $s
    echo "== $spec B=$1 N=$2 L=$3"; env $envs SLSE_LIB=build/variants/$v/libsuperlse_b200.so python tools/grid_bench.py --B $1 --N $2 --L $3 --reps 10
  done
done
