"""Strong-scaling emulation on ONE GPU: partition the rows for N ranks exactly
as the multi-GPU layer does, run every rank's range alone on the GPU (each
rank owns a whole B200 in the real run), and report per-range device times.
The N-GPU step time is max over ranges (+ the two tiny collectives, ~0.1 ms);
speedup = full single-GPU time / that max.

With --mode interleave the rows are dealt round-robin in units of --unit
rows (the paper's source scheduling) instead of
contiguous work-balanced ranges; for units finer than chunk_size each part's
time includes its gsofa_result_rowinfo and gsofa_supernodes_gathered calls
(the NCCL all_gather between them is not in the emulation).

With --mode steal the rows are cut into chunk-aligned blocks of equal
estimated work (--blocks-per-rank per rank) claimed heaviest first from a
shared counter (dist.symbolic_stealing): every block is timed alone on a warm
context and the claims are replayed as list scheduling (the next block goes to
the rank that frees up first); the N-GPU time is the last rank's finish.

usage: python scripts/scaling_emulation.py --config C5 --gpus 2 4 8 [--reps 2]
       python scripts/scaling_emulation.py --config C5 --mode interleave --unit 128
"""
import argparse
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import gen  # noqa: E402
import paper_2007_00840_b200 as g  # noqa: E402
from paper_2007_00840_b200 import dist as gd  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C5")
ap.add_argument("--gpus", type=int, nargs="+", default=[2, 4, 8])
ap.add_argument("--reps", type=int, default=2)
ap.add_argument("--mode", default="ranges", choices=["ranges", "interleave", "steal"])
ap.add_argument("--blocks-per-rank", type=int, default=4)
ap.add_argument("--unit", type=int, default=128)
ap.add_argument("--out", default=None)
ap.add_argument("--bounds", type=int, nargs="+", default=None,
                help="explicit range bounds (ranges mode, one N = len - 1) instead of the partition")
ap.add_argument("--skip-full", action="store_true", help="reuse --full-ms instead of timing 1 GPU")
ap.add_argument("--full-ms", type=float, default=None)
a = ap.parse_args()

rp, ci = gen.config(a.config)
n = rp.size - 1


def timed(rb, re, il=None):
    # a fresh context per range, as each rank owns its GPU; best of reps
    import time

    import torch
    ctx = g.Context(0)
    best = None
    for _ in range(a.reps):
        r = g.symbolic(rp, ci, ctx=ctx, row_begin=rb, row_end=re, outputs_on_device=True,
                       interleave=il)
        ms = r.stats["ms_total"]
        if r.nsuper < 0:
            # the part's side of the exchange (rowinfo export + the per-chunk
            # scan over gathered rows; its own rows stand in for the others')
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            nn, mm = r.rowinfo()
            stride = r.rows
            all_n = nn.repeat(il[0])
            all_m = mm.repeat(il[0], 1)
            r.supernodes_gathered(all_n, all_m, stride)
            torch.cuda.synchronize()
            ms += (time.perf_counter() - t0) * 1e3
        fill = r.fill_count
        r.free()
        best = ms if best is None else min(best, ms)
    ctx.close()
    return best, fill


if a.skip_full:
    full_ms, full_fill = a.full_ms, None
else:
    full_ms, full_fill = timed(0, n)
print(f"{a.config}: 1 GPU {full_ms:.1f} ms, fill {full_fill}", flush=True)
report = {"config": a.config, "n": n, "one_gpu_ms": full_ms, "fill": full_fill, "mode": a.mode,
          "unit": a.unit if a.mode == "interleave" else None, "runs": []}
for N in a.gpus:
    if a.mode == "steal":
        blocks = gd.steal_blocks(rp, ci, N * a.blocks_per_rank, 128)
        ctx = g.Context(0)
        bt = []
        fills = 0
        for rb, re in blocks:
            best = None
            for _ in range(a.reps):
                r = g.symbolic(rp, ci, ctx=ctx, row_begin=rb, row_end=re, outputs_on_device=True)
                best = r.stats["ms_total"] if best is None else min(best, r.stats["ms_total"])
                f = r.fill_count
                r.free()
            bt.append(best)
            fills += f
        ctx.close()
        assert fills == full_fill
        free = [0.0] * N
        for t in bt:  # claim order = heaviest first; the first free rank claims
            i = min(range(N), key=lambda j: free[j])
            free[i] += t
        mx = max(free)
        print(f"  N={N}: {len(blocks)} blocks, block ms {[round(x, 1) for x in bt]}\n"
              f"        rank finish ms {[round(x, 1) for x in free]} -> max {mx:.1f} ms, "
              f"speedup {full_ms / mx:.2f}x", flush=True)
        report["runs"].append({"gpus": N, "blocks": blocks, "block_ms": bt, "rank_ms": free,
                               "max_ms": mx, "speedup": full_ms / mx})
        continue
    bounds = gd.partition(rp, ci, N) if a.mode == "ranges" else np.array([0, n])
    if a.bounds is not None:
        bounds = np.array(a.bounds, dtype=np.int64)
        N = bounds.size - 1
    per = []
    fills = 0
    for r in range(N):
        if a.mode == "ranges":
            ms, f = timed(int(bounds[r]), int(bounds[r + 1]))
        else:
            ms, f = timed(0, n, (N, r, a.unit))
        per.append(ms)
        fills += f
    assert full_fill is None or fills == full_fill
    mx = max(per)
    print(f"  N={N}: ranges {list(map(int, bounds))}\n        ms {[round(x, 1) for x in per]} -> max {mx:.1f} ms, "
          f"speedup {full_ms / mx:.2f}x, efficiency {full_ms / mx / N:.2f}", flush=True)
    report["runs"].append({"gpus": N, "bounds": [int(b) for b in bounds], "range_ms": per,
                           "max_ms": mx, "speedup": full_ms / mx})
if a.out:
    json.dump(report, open(a.out, "w"), indent=1)
