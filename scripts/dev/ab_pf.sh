#!/bin/bash
# latency shape with the bulk-copy adjacency prefetch vs the throughput shape
run() { timeout 300 python scripts/probe.py "$@" 2>&1 | grep -A6 "rep 1"; }
for W in 0 1; do
  export GSOFA_SOLO_WIDE=$W
  echo "== wide=$W C4 height"; GSOFA_SRC_TRACE=/tmp/s.bin run --config C4 --schedule height --reps 2
  for S in threshold height; do
    echo "== wide=$W C5 top $S"; GSOFA_SRC_TRACE=/tmp/s.bin run --config C5 --schedule $S --reps 2 --rows 2074239:2082353
    echo "== wide=$W C5 $S"; run --config C5 --schedule $S --reps 2
    echo "== wide=$W C2 $S"; run --config C2 --schedule $S --reps 2
  done
done
