python -c "from paper_2007_00840_b200.build import build; build()"
L=paper_2007_00840_b200
timeout 600 python -m pytest tests/test_parity_gpu.py -x -q 2>&1 | tail -2
for c in C2 C3 C4 C5; do
for v in "" m1; do
  echo "== $c ${v:-base}"; GSOFA_LIB=$L/libgsofa${v:+_$v}.so timeout 120 python scripts/probe.py --config $c --reps 2 | tail -1
done; done
GSOFA_GROUP_TRACE=/tmp/t.bin timeout 120 python scripts/probe.py --config C2 --reps 1 2>&1 | head -7
