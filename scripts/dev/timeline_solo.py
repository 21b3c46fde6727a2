"""Dev: concurrency timeline of the solo kernel from GSOFA_SRC_TRACE (start/end
ns per source): active sources per time slice, and when each row band ran."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import gen  # noqa: E402
import paper_2007_00840_b200 as g  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "C5"
path = "/tmp/gsofa_src_trace.bin"
os.environ["GSOFA_SRC_TRACE"] = path
rp, ci = gen.config(cfg)
n = rp.size - 1
ctx = g.Context(0)
for _ in range(2):
    r = g.symbolic(rp, ci, ctx=ctx, outputs_on_device=True)
    ms = r.stats["ms_total"]
    r.free()
t = np.fromfile(path, dtype=np.int64).reshape(-1, 4)
solo = np.nonzero(t[:, 1])[0]
t0 = t[solo, 0].min()
st, en = (t[solo, 0] - t0) / 1e6, (t[solo, 1] - t0) / 1e6
T = en.max()
print(f"{cfg}: call {ms:.0f} ms, solo sources {solo.size} of {n}, last solo end {T:.0f} ms")
edges = np.linspace(0, T, 21)
for a, b in zip(edges[:-1], edges[1:]):
    mid = (a + b) / 2
    act = int(((st <= mid) & (en > mid)).sum())
    started = (st >= a) & (st < b)
    rows = solo[started]
    band = f"rows {rows.min()}..{rows.max()}" if rows.size else ""
    print(f"  {a:7.0f}-{b:7.0f} ms: active {act:5d}  started {int(started.sum()):6d}  {band}")
dur = en - st
for q in (50, 90, 99, 100):
    print(f"  source duration p{q}: {np.percentile(dur, q):.1f} ms")
