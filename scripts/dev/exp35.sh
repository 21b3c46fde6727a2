python -c "from paper_2007_00840_b200.build import build; build()"
for C in 0 24576 38752 0 38752; do
  echo "== C3 fifo C=$C"; timeout 300 python scripts/probe.py --config C3 --schedule fifo --C $C --reps 2 | tail -1 | cut -c1-240
done
for C in 0 32768; do
  echo "== C3-20000 fifo C=$C"; timeout 300 python scripts/probe.py --config C3 --scale 20000 --schedule fifo --C $C --reps 2 | tail -1 | cut -c1-240
done
