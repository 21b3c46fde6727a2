"""Dev: can one GPU overlap a chain-bound call (a slice of the top separator)
with a throughput-bound call (a slice of the light rows)?  Runs the two
ranges alone, then concurrently from two host threads on two contexts."""
import os
import sys
import threading
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import gen  # noqa: E402
import paper_2007_00840_b200 as g  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "C5"
N = int(sys.argv[2]) if len(sys.argv) > 2 else 8
rp, ci = gen.config(cfg)
n = rp.size - 1
top = {"C5": 16384, "C2": 4096}[cfg]
B = n - top
# rank N-1's share: the last top slice and a work-balanced slice of the bottom
b_bounds = g.partition_rows(rp[:B + 1].copy(), ci[:rp[B]].copy(), N) if False else None
sub = g.partition_rows(rp, ci, 64)  # fine split, take an eighth of the bottom work by rows
# bottom slice: rows [B - len, B) with ~1/N of the bottom estimated work
bw = np.searchsorted(sub, B)
lo = int(sub[max(0, bw - 64 // N)]) if bw > 0 else 0
ranges = [(n - top // N, n), (lo, B)]
print(cfg, "ranges", ranges, flush=True)
ctxs = [g.Context(0), g.Context(0)]


def run(i, out):
    rb, re = ranges[i]
    r = g.symbolic(rp, ci, ctx=ctxs[i], row_begin=rb, row_end=re, outputs_on_device=True)
    out[i] = (r.stats["ms_total"], r.fill_count)
    r.free()


for i in range(2):  # warm
    o = {}
    run(i, o)
alone = []
for i in range(2):
    o = {}
    torch.cuda.synchronize()
    t = time.perf_counter()
    run(i, o)
    torch.cuda.synchronize()
    alone.append((time.perf_counter() - t) * 1e3)
    print(f"range {ranges[i]} alone: wall {alone[-1]:.1f} ms, device {o[i][0]:.1f} ms", flush=True)
for rep in range(2):
    o = {}
    torch.cuda.synchronize()
    t = time.perf_counter()
    th = [threading.Thread(target=run, args=(i, o)) for i in range(2)]
    for x in th:
        x.start()
    for x in th:
        x.join()
    torch.cuda.synchronize()
    both = (time.perf_counter() - t) * 1e3
    print(f"concurrent: wall {both:.1f} ms (device {o[0][0]:.1f} / {o[1][0]:.1f}); "
          f"sum alone {sum(alone):.1f}, max alone {max(alone):.1f}", flush=True)
