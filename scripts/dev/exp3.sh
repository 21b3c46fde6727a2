python -c "from paper_2007_00840_b200.build import build; build()"
timeout 600 python -m pytest tests/test_parity_gpu.py -x -q 2>&1 | tail -3
L=paper_2007_00840_b200
for c in C2 C3 C5; do
for v in "" b2 m4 m4b2; do
  lib=$L/libgsofa${v:+_$v}.so
  echo "== $c ${v:-base}"; GSOFA_LIB=$lib timeout 120 python scripts/probe.py --config $c --reps 2 | tail -1
  echo "== $c ${v:-base} nosolo"; GSOFA_LIB=$lib GSOFA_SOLO_CTAS=0 timeout 120 python scripts/probe.py --config $c --reps 2 | tail -1
done; done
