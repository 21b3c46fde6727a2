python -c "from paper_2007_00840_b200.build import build; build()"
L=paper_2007_00840_b200
timeout 900 python -m pytest tests/test_parity_gpu.py -x -q 2>&1 | tail -2
for c in C2 C3 C4 C5; do
for v in "" nopf; do
  echo "== $c ${v:-pf}"; GSOFA_LIB=$L/libgsofa${v:+_$v}.so timeout 120 python scripts/probe.py --config $c --reps 2 | tail -1 | cut -c1-60
done; done
echo "== C4 hub rows only"; timeout 120 python scripts/probe.py --config C4 --reps 2 --rows 1584963:1585478 | tail -1 | cut -c1-60
GSOFA_LIB=$L/libgsofa_nopf.so timeout 120 python scripts/probe.py --config C4 --reps 2 --rows 1584963:1585478 | tail -1 | cut -c1-60
