python -c "from paper_2007_00840_b200.build import build; build()"
L=paper_2007_00840_b200
for c in C2 C3 C4 C5; do
  echo "== $c base"; timeout 120 python scripts/probe.py --config $c --reps 2 | tail -1
  echo "== $c m1"; GSOFA_LIB=$L/libgsofa_m1.so timeout 120 python scripts/probe.py --config $c --reps 2 | tail -1
  echo "== $c m1 solo148"; GSOFA_LIB=$L/libgsofa_m1.so GSOFA_SOLO_CTAS=148 timeout 120 python scripts/probe.py --config $c --reps 2 | tail -1
done
