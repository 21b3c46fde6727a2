L=paper_2007_00840_b200
for v in pf base pf base; do echo "== C4hubs $v"; GSOFA_LIB=$L/libgsofa_$v.so timeout 120 python scripts/probe.py --config C4 --reps 2 --rows 1584963:1585478 | tail -1 | cut -c1-60; done
for c in C2 C3 C4 C5; do for v in pf base; do
  echo "== $c $v"; GSOFA_LIB=$L/libgsofa_$v.so timeout 120 python scripts/probe.py --config $c --reps 2 | tail -1 | cut -c1-60
done; done
