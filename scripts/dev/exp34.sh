L=paper_2007_00840_b200
for c in "C3" "C3 --scale 10000" "C2 --scale 40"; do for v in 4 8 16 4 8 16; do
  echo "== $c f$v"; GSOFA_LIB=$L/libgsofa_f$v.so timeout 300 python scripts/probe.py --config $c --schedule fifo --reps 2 | tail -1 | cut -c1-70
done; done
GSOFA_LIB=$L/libgsofa_f8.so timeout 600 python -m pytest tests/test_parity_gpu.py -x -q -k "fifo or auto or C3" 2>&1 | tail -1
