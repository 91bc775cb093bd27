#!/bin/bash
# Solve times: current tree vs build/old_tree (a previous commit's package +
# library), alternating, REPS times.  CASES="cfg:B cfg:B ..."
cd "$(dirname "$0")/.."
for i in $(seq ${REPS:-2}); do
  for c in ${CASES:-2:4096 3:1024 4:256}; do
    python tools/time_root.py . ${c%%:*} ${c##*:}
    python tools/time_root.py build/old_tree ${c%%:*} ${c##*:}
  done
done
