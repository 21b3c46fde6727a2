"""Dev probe: run the CUDA path on a config and print stats (no oracle)."""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import gen  # noqa: E402
import paper_2007_00840_b200 as g  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C2")
ap.add_argument("--scale", type=int, default=None)
ap.add_argument("--reps", type=int, default=2)
ap.add_argument("--C", type=int, default=0)
ap.add_argument("--fill-first", action="store_true")
a = ap.parse_args()
t = time.time()
rp, ci = gen.config(a.config, a.scale)
print(f"{a.config} n={rp.size-1} nnz={ci.size} gen {time.time()-t:.1f}s", flush=True)
ctx = g.Context(0)
for i in range(a.reps):
    t = time.time()
    r = g.symbolic(rp, ci, ctx=ctx, max_concurrent=a.C, fill_first=a.fill_first, outputs_on_device=True)
    dt = time.time() - t
    s = r.stats
    print(f"rep {i}: wall {dt*1e3:.1f} ms  dev {s['ms_total']:.1f} ms  trav {s['ms_traverse']:.1f} "
          f"ext {s['ms_extract']:.1f} sn {s['ms_supernode']:.2f} | fill {r.fill_count} nnzL {r.nnz_L} "
          f"nnzU {r.nnz_U} nsuper {r.nsuper} | edges {s['edge_inspections']:.3e} items {s['frontier_items']:.3e} "
          f"rounds {s['rounds']} batches {s['batches']} C {s['max_batch']} launches {s['kernel_launches']}",
          flush=True)
    r.free()
