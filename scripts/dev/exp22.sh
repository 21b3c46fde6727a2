python -c "from paper_2007_00840_b200.build import build; build()"
for a in 0.97 0.94 0.90; do
  echo "== C5 alpha $a"; GSOFA_PART_ALPHA=$a timeout 900 python scripts/scaling_emulation.py --config C5 --gpus 8 | tail -2
done
for a in 0.94 0.90; do
  echo "== C2 alpha $a"; GSOFA_PART_ALPHA=$a timeout 900 python scripts/scaling_emulation.py --config C2 --gpus 8 | tail -2
done
