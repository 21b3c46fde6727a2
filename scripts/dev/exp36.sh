python -c "from paper_2007_00840_b200.build import build; build()"
for r in 2092539:2097152 2087915:2092539 2076464:2083281; do for sch in threshold fifo; do
  echo "== C5 $r $sch"; timeout 600 python scripts/probe.py --config C5 --rows $r --schedule $sch --reps 2 | tail -1 | cut -c1-240
done; done
for r in 261027:262144 258777:259905; do for sch in threshold fifo; do
  echo "== C2 $r $sch"; timeout 600 python scripts/probe.py --config C2 --rows $r --schedule $sch --reps 2 | tail -1 | cut -c1-240
done; done
