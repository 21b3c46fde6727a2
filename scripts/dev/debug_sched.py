"""Dev: failure map of both schedules on random graphs vs the oracle."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
import gen, oracle
import paper_2007_00840_b200 as g
ctx = g.Context(0)
for seed in range(12):
    rng = np.random.default_rng(seed)
    n = int(rng.integers(1, 300)); d = float(rng.uniform(0.005, 0.2))
    rp, ci = gen.random_graph(n, d, seed=100 + seed)
    want = oracle.symbolic(rp, ci)
    line = []
    for sch in ("threshold", "fifo"):
        for mc in (0, 32, 64):
            for ff in (0, 1):
                r = g.symbolic(rp, ci, ctx=ctx, schedule=sch, max_concurrent=mc, fill_first=bool(ff))
                a = r.to_numpy()
                ok = np.array_equal(a["L_colidx"], want["L_colidx"]) and np.array_equal(a["U_colidx"], want["U_colidx"])
                if not ok:
                    Lp = a["L_rowptr"]; bad = np.nonzero(Lp != want["L_rowptr"])[0]
                    line.append(f"{sch[0]}{mc}{'f' if ff else ''}:BAD(row{bad[0]-1 if bad.size else -1},L{r.nnz_L}/{want['nnz_L']},rounds{r.stats['rounds']},b{r.stats['batches']})")
                r.free()
    print(seed, n, round(d, 3), "OK" if not line else " ".join(line), flush=True)
# fresh context per call
for seed in (2,):
    rng = np.random.default_rng(seed)
    n = int(rng.integers(1, 300)); d = float(rng.uniform(0.005, 0.2))
    rp, ci = gen.random_graph(n, d, seed=100 + seed)
    want = oracle.symbolic(rp, ci)
    for mc in (32, 64, 0):
        r = g.symbolic(rp, ci, schedule="fifo", max_concurrent=mc)
        print("fresh ctx fifo mc", mc, r.nnz_L, want["nnz_L"], r.stats["rounds"], r.stats["batches"])
        r.free()
