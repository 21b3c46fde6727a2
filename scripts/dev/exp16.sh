python -c "from paper_2007_00840_b200.build import build; build()"
for sc in 74 148 296; do for lc in 300 100000; do
  echo "== C5 solo $sc light $lc"; GSOFA_SOLO_CTAS=$sc GSOFA_LIGHT_CTAS=$lc timeout 120 python scripts/probe.py --config C5 --reps 2 | tail -1 | cut -c1-60
done; done
