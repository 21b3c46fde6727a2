python -c "from paper_2007_00840_b200.build import build; build()"
for c in "C1" "C3 --scale 10000" "C3 --scale 20000" "C4 --scale 300" "C5 --scale 40"; do
  for m in "--schedule fifo" "--schedule threshold"; do
    echo "== $c $m"; timeout 300 python scripts/probe.py --config $c $m --reps 3 | tail -1 | cut -c1-200
  done
done
python -c "
import gen, numpy as np
for nm, sc in [('C1',None),('C2',None),('C3',None),('C3',10000),('C4',300),('C5',40),('C2',40)]:
    rp, ci = gen.config(nm, sc); n = rp.size-1
    rows = np.repeat(np.arange(n), np.diff(rp))
    bw = np.abs(rows - ci).max(); p99 = np.percentile(np.abs(rows-ci), 99)
    print(nm, sc, 'n', n, 'bandwidth', bw, 'bw/n %.3f' % (bw/n), 'p99/n %.4f' % (p99/n))
"
