python -c "from paper_2007_00840_b200.build import build; build()"
L=paper_2007_00840_b200
for c in C2 C3 C4 C5; do
for v in "" b1 b3; do
  echo "== $c ${v:-b2}"; GSOFA_LIB=$L/libgsofa${v:+_$v}.so timeout 120 python scripts/probe.py --config $c --reps 2 | tail -1 | cut -c1-60
done; done
timeout 900 python -m pytest tests/test_parity_gpu.py -x -q 2>&1 | tail -2
