#!/bin/bash
# solo kernel shape A/B (GSOFA_SOLO_WIDE) x threshold order, full configs and
# the chain-bound top ranges of an 8-way C5 split
run() { timeout 300 python scripts/probe.py "$@" 2>&1 | grep "rep 1"; }
for W in 0 1; do
  for S in threshold height; do
    echo "== wide=$W $S"
    export GSOFA_SOLO_WIDE=$W
    run --config C4 --schedule $S --reps 2
    run --config C2 --schedule $S --reps 2
    run --config C5 --schedule $S --reps 2 --rows 2074239:2082353
    run --config C5 --schedule $S --reps 2 --rows 2092230:2097152
    run --config C5 --schedule $S --reps 2
  done
done
