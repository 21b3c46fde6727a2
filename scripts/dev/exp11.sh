python -c "from paper_2007_00840_b200.build import build; build()"
L=paper_2007_00840_b200
for c in C2 C3 C4 C5; do
  echo "== $c base"; timeout 120 python scripts/probe.py --config $c --reps 2 | tail -1
  echo "== $c f1"; GSOFA_LIB=$L/libgsofa_f1.so timeout 120 python scripts/probe.py --config $c --reps 2 | tail -1
done
GSOFA_LIB=$L/libgsofa_f1.so timeout 600 python -m pytest tests/test_parity_gpu.py -x -q 2>&1 | tail -2
