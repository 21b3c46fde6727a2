L=paper_2007_00840_b200
GSOFA_LIB=$L/libgsofa_few.so timeout 600 python -m pytest tests/test_parity_gpu.py -x -q 2>&1 | tail -1
for v in few base few base; do echo "== C5top256 $v"; GSOFA_LIB=$L/libgsofa_$v.so timeout 200 python scripts/probe.py --config C5 --reps 2 --rows 2096896:2097152 | tail -1 | cut -c1-60; done
for v in few base; do echo "== C4hubs $v"; GSOFA_LIB=$L/libgsofa_$v.so timeout 200 python scripts/probe.py --config C4 --reps 2 --rows 1584963:1585478 | tail -1 | cut -c1-60; done
for c in C2 C4 C5; do for v in few base few base; do
  echo "== $c $v"; GSOFA_LIB=$L/libgsofa_$v.so timeout 120 python scripts/probe.py --config $c --reps 2 | tail -1 | cut -c1-60
done; done
