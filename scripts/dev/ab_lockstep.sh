#!/bin/bash
# lockstep-only (every group on the 32-source lockstep kernel, no solo) vs the
# default routing, on the chain-bound C5 top ranges, C2 and C4; group traces
run() { timeout 300 python scripts/probe.py "$@" 2>&1 | grep -A12 "rep 1"; }
for R in 2074239:2082353 2092230:2097152; do
  echo "== C5 rows $R default"; run --config C5 --schedule threshold --reps 2 --rows $R
  echo "== C5 rows $R lockstep only"; GSOFA_SOLO_CTAS=0 GSOFA_GROUP_TRACE=/tmp/g.bin run --config C5 --schedule threshold --reps 2 --rows $R
done
echo "== C2 lockstep only"; GSOFA_SOLO_CTAS=0 GSOFA_GROUP_TRACE=/tmp/g.bin run --config C2 --schedule threshold --reps 2
echo "== C5 lockstep only"; GSOFA_SOLO_CTAS=0 GSOFA_GROUP_TRACE=/tmp/g.bin run --config C5 --schedule threshold --reps 2
echo "== C4 height wide"; GSOFA_SOLO_WIDE=1 GSOFA_SRC_TRACE=/tmp/s.bin run --config C4 --schedule height --reps 2
