#!/bin/bash
# the current library vs round 1's (GSOFA_LIB) on the same box, id order
for i in 1 2; do
  for L in paper_2007_00840_b200/libgsofa.so paper_2007_00840_b200/libgsofa_r1ref.so; do
    echo "== $L"
    for C in C5 C2 C4; do
      GSOFA_LIB=$L timeout 300 python scripts/probe.py --config $C --schedule threshold --reps 3 2>&1 | grep "rep 2" | cut -c1-80
    done
  done
done
