#!/bin/bash
# A/B of the threshold orders (id vs etree height) on the full configs
for C in C2 C4 C5; do
  for S in threshold height; do
    timeout 300 python scripts/probe.py --config $C --schedule $S --reps 3 2>&1 | tail -2
  done
done
