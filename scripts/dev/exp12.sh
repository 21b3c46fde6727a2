python -c "from paper_2007_00840_b200.build import build; build()"
for c in C2 C3 C4 C5; do
  for cfg in "" "GSOFA_ABORT_MS=1" "GSOFA_ABORT_MS=20" "GSOFA_SOLO_TOP=100000" "GSOFA_SOLO_TOP=600"; do
    echo "== $c ${cfg:-default}"; env $cfg timeout 120 python scripts/probe.py --config $c --reps 2 | tail -1 | sed 's/|.*edges/| edges/'
  done
done
