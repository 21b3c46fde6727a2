python -c "from paper_2007_00840_b200.build import build; build()"
for c in C4 C1 C2; do
  for cfg in "" "GSOFA_SOLO_TOP=100000" "" "GSOFA_SOLO_TOP=100000"; do
    echo "== $c ${cfg:-default}"; env $cfg timeout 120 python scripts/probe.py --config $c --reps 3 | tail -1 | cut -c1-60
  done
done
for r in 2092539:2097152 1046157:1691321; do for cfg in "" "GSOFA_SOLO_TOP=100000"; do
  echo "== C5 rows $r ${cfg:-default}"; env $cfg timeout 120 python scripts/probe.py --config C5 --reps 2 --rows $r | tail -1 | cut -c1-60
done; done
