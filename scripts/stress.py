"""Repeat every config several times in one context with checked mode on:
results must be identical call to call (a race in the traversal would show
up as a changed count or a failed audit).  Run with GSOFA_CHECK_CLEAN=1 to
also verify that every workspace slot is zero again after each call.

usage: python scripts/stress.py [--reps 4]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import gen  # noqa: E402
import paper_2007_00840_b200 as g  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--reps", type=int, default=4)
ap.add_argument("--configs", nargs="+", default=["C1", "C3", "C2", "C4", "C5"])
a = ap.parse_args()
ctx = g.Context(0)
for name in a.configs:
    rp, ci = gen.config(name)
    ref = None
    for i in range(a.reps):
        r = g.symbolic(rp, ci, ctx=ctx, outputs_on_device=True, checked=True)
        key = (r.fill_count, r.nnz_L, r.nnz_U, r.nsuper)
        ms = r.stats["ms_total"]
        r.free()
        if ref is None:
            ref = key
        assert key == ref, (name, i, key, ref)
        print(f"{name} rep {i}: {ms:.1f} ms {key}", flush=True)
print("stress ok")
