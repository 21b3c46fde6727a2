python -c "from paper_2007_00840_b200.build import build; build()"
L=paper_2007_00840_b200

for c in C2 C3 C4 C5; do
for v in m3b1 m4b1 m4b2 m3b1; do
  echo "== $c $v"; GSOFA_LIB=$L/libgsofa_$v.so timeout 120 python scripts/probe.py --config $c --reps 2 | tail -1 | cut -c1-60
done; done
