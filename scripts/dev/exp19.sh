L=paper_2007_00840_b200
timeout 900 python -m pytest tests/test_parity_gpu.py -x -q 2>&1 | tail -1
for v in fast base; do echo "== top-range $v"; GSOFA_LIB=$L/libgsofa_$v.so timeout 120 python scripts/probe.py --config C2 --reps 2 --rows 259905:261027 | tail -1 | cut -c1-60; done
for v in fast base; do echo "== C4 hubs $v"; GSOFA_LIB=$L/libgsofa_$v.so timeout 120 python scripts/probe.py --config C4 --reps 2 --rows 1584963:1585478 | tail -1 | cut -c1-60; done
for c in C2 C3 C4 C5; do
for v in fast base fast base; do
  echo "== $c $v"; GSOFA_LIB=$L/libgsofa_$v.so timeout 120 python scripts/probe.py --config $c --reps 2 | tail -1 | cut -c1-60
done; done
