"""Memory-budget and chunk-size sweeps.

For each traversal-arena budget ("reduce the number of concurrent
sources" until the working set fits), run the full factorization and check
that the output is identical to the unconstrained run: same counts, same
supernodes and the same 64-bit checksum of the L/U column arrays, computed
on the GPU.  Then sweep chunk_size (maximum supernode size)
and report nsuper and time.

With --schedule fifo the sweep also reports the external frontier spill
(queue items written to host memory).

usage: python scripts/budget_sweep.py --config C5 --budgets-gb 1 5 16 0
       python scripts/budget_sweep.py --config C3 --schedule fifo --budgets-gb 1 5 16 0
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import gen  # noqa: E402
import paper_2007_00840_b200 as g  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C5")
ap.add_argument("--budgets-gb", type=float, nargs="+", default=[1, 5, 16, 0])
ap.add_argument("--chunks", type=int, nargs="+", default=[64, 128, 256])
ap.add_argument("--schedule", default="auto", choices=["auto", "threshold", "fifo", "height"])
ap.add_argument("--out", default=None)
a = ap.parse_args()

import torch  # noqa: E402

rp, ci = gen.config(a.config)


def checksum(t):
    # position-weighted sum mod 2^61-1, computed on the GPU in int64 chunks
    m = (1 << 61) - 1
    acc = 0
    step = 1 << 26
    for i in range(0, t.numel(), step):
        x = t[i:i + step].to(torch.int64)
        w = torch.arange(i + 1, i + 1 + x.numel(), device=x.device, dtype=torch.int64) % 1000003
        acc = (acc + int(((x * w) % m).sum().item())) % m
    return acc


def run(budget_gb=0.0, chunk=128):
    ctx = g.Context(0, int(budget_gb * (1 << 30)))
    best = None
    for _ in range(2):
        r = g.symbolic(rp, ci, ctx=ctx, chunk_size=chunk, outputs_on_device=True,
                       schedule=a.schedule)
        ms = r.stats["ms_total"]
        best = ms if best is None else min(best, ms)
        keep = r
        if _ == 0:
            r.free()
    t = keep.to_torch()
    info = dict(budget_gb=budget_gb, chunk=chunk, ms=best, fill=keep.fill_count, nsuper=keep.nsuper,
                nnz_L=keep.nnz_L, nnz_U=keep.nnz_U, concurrent_sources=keep.stats["max_batch"],
                batches=keep.stats["batches"], frontier_spilled=keep.stats["frontier_spilled"],
                schedule=keep.schedule,
                sum_L=checksum(t["L_colidx"]), sum_U=checksum(t["U_colidx"]),
                sum_sn=checksum(t["sn_start"]))
    keep.free()
    ctx.close()
    del t
    torch.cuda.empty_cache()
    return info


rows = []
for b in a.budgets_gb:
    rows.append(run(b))
    print(json.dumps(rows[-1]), flush=True)
ref = rows[-1]
for r in rows:
    same = all(r[k] == ref[k] for k in ("fill", "nsuper", "nnz_L", "nnz_U", "sum_L", "sum_U", "sum_sn"))
    print(f"budget {r['budget_gb'] or 'auto':>5} GB: {r['ms']:9.1f} ms, {r['concurrent_sources']:6d} concurrent "
          f"sources, {r['batches']} batches, {r['frontier_spilled']} frontier items spilled to host, "
          f"identical to the unconstrained run: {same}")
    assert same
chunks = [run(0, c) for c in a.chunks]
for c in chunks:
    print(f"chunk_size {c['chunk']:4d}: nsuper {c['nsuper']}, {c['ms']:.1f} ms "
          f"(L/U identical: {c['sum_L'] == ref['sum_L'] and c['sum_U'] == ref['sum_U']})")
if a.out:
    json.dump({"config": a.config, "budgets": rows, "chunks": chunks}, open(a.out, "w"), indent=1)
