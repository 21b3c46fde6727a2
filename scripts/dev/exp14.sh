python -c "from paper_2007_00840_b200.build import build; build()"
for a in 1.0 1.04 1.08; do
  echo "== alpha $a"; GSOFA_PART_ALPHA=$a timeout 900 python scripts/scaling_emulation.py --config C5 --gpus 8 | tail -2
done
for a in 1.0 1.08; do
  echo "== C4 alpha $a"; GSOFA_PART_ALPHA=$a timeout 900 python scripts/scaling_emulation.py --config C4 --gpus 8 | tail -2
done
