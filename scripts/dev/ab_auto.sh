#!/bin/bash
# AUTO (tree-shape choice of the threshold order) vs explicit orders, and the
# current library vs round 1's on the same box
for i in 1 2; do
  for L in paper_2007_00840_b200/libgsofa.so paper_2007_00840_b200/libgsofa_r1ref.so; do
    echo "== $L threshold"
    for C in C5 C2 C4; do
      GSOFA_LIB=$L timeout 300 python scripts/probe.py --config $C --schedule threshold --reps 3 2>&1 | grep "rep 2" | cut -c1-80
    done
  done
done
echo "== auto"
for C in C5 C2 C4 C1 C3; do
  GSOFA_TIMELINE=1 timeout 300 python scripts/probe.py --config $C --reps 3 2>&1 | grep "rep 2" | cut -c1-100
done
