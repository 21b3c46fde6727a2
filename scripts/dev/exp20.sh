python -c "from paper_2007_00840_b200.build import build; build()"
GSOFA_ELL=1 timeout 600 python -m pytest tests/test_parity_gpu.py -x -q 2>&1 | tail -1
for e in 1 0 1 0; do echo "== top-range ell=$e"; GSOFA_ELL=$e timeout 120 python scripts/probe.py --config C2 --reps 2 --rows 259905:261027 | tail -1 | cut -c1-60; done
for e in 1 0; do echo "== C4 hubs ell=$e"; GSOFA_ELL=$e timeout 120 python scripts/probe.py --config C4 --reps 2 --rows 1584963:1585478 | tail -1 | cut -c1-60; done
for e in 1 0; do echo "== C5 top ell=$e"; GSOFA_ELL=$e timeout 120 python scripts/probe.py --config C5 --reps 2 --rows 2092539:2097152 | tail -1 | cut -c1-60; done
for e in 1 0; do echo "== C2 full ell=$e"; GSOFA_ELL=$e timeout 120 python scripts/probe.py --config C2 --reps 2 | tail -1 | cut -c1-60; done
