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
ap.add_argument("--schedule", default="auto", choices=["auto", "threshold", "fifo", "height"])
ap.add_argument("--rows", type=str, default=None, help="row range b:e")
a = ap.parse_args()
t = time.time()
rp, ci = gen.config(a.config, a.scale)
print(f"{a.config} n={rp.size-1} nnz={ci.size} gen {time.time()-t:.1f}s", flush=True)
ctx = g.Context(0)
for i in range(a.reps):
    t = time.time()
    rb, re_ = (int(x) for x in a.rows.split(":")) if a.rows else (0, -1)
    r = g.symbolic(rp, ci, ctx=ctx, max_concurrent=a.C, fill_first=a.fill_first, outputs_on_device=True,
                   row_begin=rb, row_end=re_, schedule=a.schedule)
    dt = time.time() - t
    s = r.stats
    print(f"rep {i} [{r.schedule}]: wall {dt*1e3:.1f} ms  dev {s['ms_total']:.1f} ms  trav {s['ms_traverse']:.1f} "
          f"ext {s['ms_extract']:.1f} sn {s['ms_supernode']:.2f} | fill {r.fill_count} nnzL {r.nnz_L} "
          f"nnzU {r.nnz_U} nsuper {r.nsuper} | edges {s['edge_inspections']:.3e} items {s['frontier_items']:.3e} "
          f"rounds {s['rounds']} batches {s['batches']} C {s['max_batch']} launches {s['kernel_launches']}",
          flush=True)
    r.free()
if os.environ.get("GSOFA_GROUP_TRACE"):
    import numpy as np
    t = np.fromfile(os.environ["GSOFA_GROUP_TRACE"], dtype=np.int64).reshape(-1, 8)
    ms = t[:, 3] / 1.965e6
    order = np.argsort(-ms)
    print("groups", t.shape[0], "sum group-ms", ms.sum(), "mean", ms.mean())
    print("top groups: g steps levels items pairs | ms total (traverse, extract, cleanup)")
    for g_ in order[:10]:
        tt, te = t[g_, 4] / 1.965e6, t[g_, 5] / 1.965e6
        print(f"  g={g_} steps={t[g_,0]} levels={t[g_,1]} items={t[g_,2]} pairs={t[g_,6]} | "
              f"{ms[g_]:.2f} ({tt:.2f}, {te:.2f}, {ms[g_]-tt-te:.2f})  us/level={t[g_,4]/1.965e3/max(1,t[g_,1]):.1f} "
              f"ns/pair={t[g_,4]/1.965/max(1,t[g_,6]):.0f}")
    for q in (50, 90, 99, 99.9):
        print(f"  p{q}: ms={np.percentile(ms, q):.3f} steps={np.percentile(t[:,0], q):.0f} levels={np.percentile(t[:,1], q):.0f}")
    print(f"  sum traverse ms {t[:,4].sum()/1.965e6:.0f}  extract ms {t[:,5].sum()/1.965e6:.0f}  total {ms.sum():.0f}")
if os.environ.get("GSOFA_SRC_TRACE"):
    import numpy as np
    t = np.fromfile(os.environ["GSOFA_SRC_TRACE"], dtype=np.int64).reshape(-1, 4)
    solo = np.nonzero(t[:, 1])[0]
    if solo.size:
        t0 = t[solo, 0].min()
        dur = (t[solo, 1] - t[solo, 0]) / 1e6
        order = solo[np.argsort(-dur)]
        print(f"solo sources {solo.size}; last end {(t[solo, 1].max() - t0) / 1e6:.1f} ms after the first start")
        print("top sources: row  start_ms  dur_ms  steps  levels  us/level")
        for r in order[:12]:
            d = (t[r, 1] - t[r, 0]) / 1e6
            print(f"  {r:8d} {(t[r, 0] - t0) / 1e6:9.2f} {d:8.2f} {t[r, 2]:7d} {t[r, 3]:8d} "
                  f"{1e3 * d / max(1, t[r, 3]):8.2f}")
