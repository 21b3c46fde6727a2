python -c "from paper_2007_00840_b200.build import build; build()"
for c in C2 C5 C3; do
  for cfg in "" "GSOFA_LIGHT_CTAS=148" "GSOFA_LIGHT_CTAS=296" "GSOFA_LIGHT_CTAS=444" "GSOFA_SOLO_TOP=100000"; do
    echo "== $c ${cfg:-default}"; env $cfg timeout 120 python scripts/probe.py --config $c --reps 2 | tail -1 | cut -c1-60
  done
done
