"""Dev: repeated calls on one context vs the oracle."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
import gen, oracle
import paper_2007_00840_b200 as g
ctx = g.Context(0)
rp, ci = gen.config("C4", 60)
want = oracle.symbolic(rp, ci)
for it in range(5):
    r = g.symbolic(rp, ci, ctx=ctx)
    a = r.to_numpy()
    ok = np.array_equal(a["L_rowptr"], want["L_rowptr"]) and np.array_equal(a["U_colidx"], want["U_colidx"])
    Lp = a["L_rowptr"]; bad = np.nonzero(Lp != want["L_rowptr"])[0]
    print(os.environ.get("TAG"), "call", it, "ok" if ok else f"BAD first row {bad[0]-1 if bad.size else '?'} nnzL {r.nnz_L}/{want['nnz_L']}", flush=True)
    r.free()
