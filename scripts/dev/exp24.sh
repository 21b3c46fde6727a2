python -c "from paper_2007_00840_b200.build import build; build()"
python -c "
import torch; p=torch.cuda.get_device_properties(0); print('L2', p.L2_cache_size)"
for e in 0 1 0 1; do
  if [ $e = 1 ]; then export GSOFA_NO_PERSIST=1; else unset GSOFA_NO_PERSIST; fi
  echo "== C5top nopersist=$e"; timeout 120 python scripts/probe.py --config C5 --reps 2 --rows 2092539:2097152 | tail -1 | cut -c1-60
done
for c in C2 C3 C4 C5; do for e in 0 1; do
  if [ $e = 1 ]; then export GSOFA_NO_PERSIST=1; else unset GSOFA_NO_PERSIST; fi
  echo "== $c nopersist=$e"; timeout 120 python scripts/probe.py --config $c --reps 2 | tail -1 | cut -c1-60
done; done
unset GSOFA_NO_PERSIST
timeout 600 python -m pytest tests/test_parity_gpu.py -x -q 2>&1 | tail -1
