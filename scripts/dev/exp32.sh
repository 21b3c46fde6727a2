python -c "from paper_2007_00840_b200.build import build; build()"
for c in "C3" "C2 --scale 40" "C2"; do
  for m in "--schedule fifo" "--schedule fifo --fill-first" "--schedule threshold"; do
    echo "== $c $m"; timeout 300 python scripts/probe.py --config $c $m --reps 2 | tail -1 | cut -c1-200
  done
done
