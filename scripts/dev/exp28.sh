python -c "from paper_2007_00840_b200.build import build; build()"
for r in 2096896:2097152 2096128:2097152 2094080:2097152 2092539:2097152 2088960:2097152; do
  echo "== C5 rows $r"; timeout 200 python scripts/probe.py --config C5 --reps 2 --rows $r | tail -1 | cut -c1-60
done
