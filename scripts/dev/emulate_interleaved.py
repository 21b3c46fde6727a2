"""Emulate the interleaved multi-GPU split (NEXT-2) on one GPU: every rank
owns one contiguous light range and one chunk-aligned slice of the heavy top
rows; a rank's two ranges run concurrently (two contexts, two host threads),
the rank's time is the wall time of the pair.  Compare with the contiguous
split (one range per rank)."""
import argparse
import os
import sys
import threading
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import gen  # noqa: E402
import paper_2007_00840_b200 as g  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C5")
ap.add_argument("--gpus", type=int, default=8)
ap.add_argument("--heavy-frac", type=float, nargs="+", default=[0.3, 0.5])
ap.add_argument("--schedule", default="threshold")
a = ap.parse_args()
rp, ci = gen.config(a.config)
n = rp.size - 1
ctxs = [g.Context(0), g.Context(0)]


def run(ctx, rb, re, out, k):
    t = time.perf_counter()
    r = g.symbolic(rp, ci, ctx=ctx, row_begin=rb, row_end=re, outputs_on_device=True,
                   schedule=a.schedule)
    out[k] = (time.perf_counter() - t, r.fill_count, r.stats["ms_total"])
    r.free()


def pair(ranges):
    out = [None] * len(ranges)
    th = [threading.Thread(target=run, args=(ctxs[k], rb, re, out, k)) for k, (rb, re) in enumerate(ranges)]
    t = time.perf_counter()
    for x in th:
        x.start()
    for x in th:
        x.join()
    return time.perf_counter() - t, out


for _ in range(2):
    full_t, o = pair([(0, n)])
full_fill = o[0][1]
print(f"1 GPU: {full_t * 1e3:.1f} ms wall, dev {o[0][2]:.1f} ms, fill {full_fill}")
fine = g.partition_rows(rp, ci, 4096)
N = a.gpus
for f in a.heavy_frac:
    k0 = int(round(4096 * (1 - f)))
    h0 = int(fine[k0]) // 128 * 128
    light = [int(fine[int(round(k0 * r / N))]) for r in range(N)] + [h0]
    light[0] = 0
    heavy = [h0] + [min(n, int(fine[k0 + int(round((4096 - k0) * r / N))]) // 128 * 128) for r in range(1, N)] + [n]
    times, fills = [], 0
    for r in range(N):
        rngs = [(light[r], light[r + 1]), (heavy[r], heavy[r + 1])]
        rngs = [x for x in rngs if x[1] > x[0]]
        best = None
        for _ in range(2):
            t, o = pair(rngs)
            best = t if best is None else min(best, t)
        fills += sum(x[1] for x in o)
        times.append(best * 1e3)
    print(f"heavy_frac {f}: h0 {h0} light {light} heavy {heavy}\n  rank ms {[round(x) for x in times]} "
          f"max {max(times):.0f} -> speedup {full_t * 1e3 / max(times):.2f}x  fill ok {fills == full_fill}")
