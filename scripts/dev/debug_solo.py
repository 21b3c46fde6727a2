"""Dev: which rows differ from the oracle under lockstep-only / solo-forced / default."""
import os, sys, subprocess
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
import gen, oracle
mode = sys.argv[1] if len(sys.argv) > 1 else "default"
import paper_2007_00840_b200 as g
for name, scale in [("C4", 60), ("C4", 40), ("C2", 12)]:
    rp, ci = gen.config(name, scale)
    want = oracle.symbolic(rp, ci)
    r = g.symbolic(rp, ci)
    a = r.to_numpy()
    n = rp.size - 1
    bad = []
    for i in range(n):
        gl = a["L_colidx"][a["L_rowptr"][i]:a["L_rowptr"][i+1]]
        wl = want["L_colidx"][want["L_rowptr"][i]:want["L_rowptr"][i+1]]
        gu = a["U_colidx"][a["U_rowptr"][i]:a["U_rowptr"][i+1]]
        wu = want["U_colidx"][want["U_rowptr"][i]:want["U_rowptr"][i+1]]
        if not (np.array_equal(gl, wl) and np.array_equal(gu, wu)):
            bad.append((i, gl.size, wl.size, gu.size, wu.size))
    print(mode, name, scale, "n", n, "bad rows", len(bad), bad[:8], "groups of bad:", sorted(set(b[0]//32 for b in bad))[:20], flush=True)
