#!/bin/bash
# A/B of the threshold orders (id vs etree height) on the full configs;
# GSOFA_TIMELINE prints the per-phase times of a call
CFGS=${CFGS:-"C2 C4 C5"}
for C in $CFGS; do
  for S in threshold height; do
    timeout 300 python scripts/probe.py --config $C --schedule $S --reps 3 2>&1 | tail -2
  done
done
