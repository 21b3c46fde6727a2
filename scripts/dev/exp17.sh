L=paper_2007_00840_b200
timeout 900 python -m pytest tests/test_parity_gpu.py -x -q 2>&1 | tail -2
for c in C2 C3 C4 C5; do
for v in ell0 base ell0 base; do
  echo "== $c $v"; GSOFA_LIB=$L/libgsofa_$v.so timeout 120 python scripts/probe.py --config $c --reps 2 | tail -1 | cut -c1-60
done; done
