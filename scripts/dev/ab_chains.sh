#!/bin/bash
# chain-bound row ranges (the top ranks of an 8-way C5 split, C4 whole) in
# both threshold orders, with the per-source solo trace
for S in threshold height; do
  GSOFA_SRC_TRACE=/tmp/src.bin timeout 300 python scripts/probe.py --config C4 --schedule $S --reps 2 2>&1 | tail -16
  for R in 2074239:2082353 2092230:2097152; do
    GSOFA_SRC_TRACE=/tmp/src.bin timeout 300 python scripts/probe.py --config C5 --schedule $S --reps 2 --rows $R 2>&1 | tail -16
  done
done
