"""Pins the reading of the paper's fine-grained max-id relaxation (fig:alg is a
placeholder; the rules are reconstructed from the prose, R2-R4)
that the CUDA traversal implements:

  R2  newMaxId = max(maxId(u), u)                         (trace values)
  R3  direct neighbours of src start at -1 ("0" in P:548) and are in the
      structure
  R4  for a neighbour w < src: atomicMin(maxId(w), newMaxId); if it lowered
      maxId(w) and w was not yet in the structure, enqueue w, and if
      newMaxId < w, (src, w) is a new fill ("5 will not be
      enqueued"); w > src is an entry of U(src, :); line 9.5
      skips the atomicMin for w already in the structure.

This is a test-side model (pure Python), not the oracle: it is pinned to the
paper's trace for src = 8 and shown to reach the oracle's
(fill2) structure on random graphs for every processing order.
"""
import json
import os

import numpy as np
import pytest

import gen
import oracle

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "paper_example.json")


def relax_source(rp, ci, src, fill_first=False, jacobi=False, rng=None, trace=None):
    n = rp.size - 1
    INF = n
    maxid = np.full(n, INF, dtype=np.int64)
    instruct = set()
    frontier = []
    for w in ci[rp[src]:rp[src + 1]].tolist():
        if w == src:
            continue
        instruct.add(w)
        if w < src:
            maxid[w] = -1
            frontier.append(w)
    while frontier:
        if trace is not None:
            trace.append(dict(frontier=sorted(frontier), maxid=maxid.copy(),
                              instruct=set(instruct)))
        order = list(frontier)
        if rng is not None:
            rng.shuffle(order)
        snap = maxid.copy()
        nxt = []
        for u in order:
            c = max((snap if jacobi else maxid)[u], u)          # R2
            for w in ci[rp[u]:rp[u + 1]].tolist():
                if w == src:
                    continue
                if w > src:
                    instruct.add(w)                             # U entry
                    continue
                if fill_first and w in instruct:                # line 9.5
                    continue
                old = maxid[w]
                if c < old:                                     # atomicMin lowered it
                    maxid[w] = c
                    if not old < w:                             # not yet in structure
                        nxt.append(w)
                        if c < w:
                            instruct.add(w)                     # new fill (L)
        frontier = sorted(set(nxt))
    if trace is not None:
        trace.append(dict(frontier=[], maxid=maxid.copy(), instruct=set(instruct)))
    return sorted(instruct)


def test_paper_trace_src8():
    g = json.load(open(GOLDEN))["trace_src8"]
    rp, ci = gen.paper_example()
    tr = []
    relax_source(rp, ci, 8, trace=tr)
    A8 = set(ci[rp[8]:rp[9]].tolist())
    assert tr[0]["frontier"] == g["iter1_frontier"]
    assert tr[1]["frontier"] == g["iter2_frontier"]
    assert tr[2]["frontier"] == g["iter3_frontier"]
    assert tr[3]["frontier"] == g["iter4_frontier"]
    for v, m in g["iter1_maxid"].items():
        assert tr[1]["maxid"][int(v)] == m          # state after iteration 1
    assert sorted(tr[1]["instruct"] - A8) == g["iter1_fills"]
    for v, m in g["iter2_maxid"].items():
        assert tr[2]["maxid"][int(v)] == m          # state after iteration 2
    assert sorted(tr[2]["instruct"] - tr[1]["instruct"]) == g["iter2_fills"]


def test_line95_skips_lowering_filled_vertex():
    """with line 9.5 maxId(5) is not lowered from 2 to 1."""
    rp, ci = gen.paper_example()
    tr = []
    relax_source(rp, ci, 8, fill_first=True, trace=tr)
    assert tr[2]["maxid"][5] == 2
    tr2 = []
    relax_source(rp, ci, 8, fill_first=False, trace=tr2)
    assert tr2[2]["maxid"][5] == 1


@pytest.mark.parametrize("seed", range(80))
def test_relaxation_reaches_oracle(seed):
    rng = np.random.default_rng(seed)
    n = int(rng.integers(8, 70))
    rp, ci = gen.random_graph(n, float(rng.uniform(0.02, 0.2)), seed=8000 + seed)
    r = oracle.rows(rp, ci)
    for src in range(n):
        want = sorted(set(r["L_colidx"][r["L_rowptr"][src]:r["L_rowptr"][src + 1]].tolist())
                      | set(r["U_colidx"][r["U_rowptr"][src] + 1:r["U_rowptr"][src + 1]].tolist()))
        for ff in (False, True):
            for jac in (False, True):
                got = relax_source(rp, ci, src, fill_first=ff, jacobi=jac,
                                   rng=np.random.default_rng(seed * 131 + src))
                assert got == want, (src, ff, jac)


# ---------------------------------------------------------------- R18
# Height order (GSOFA_SCHEDULE_HEIGHT, csrc/order.cu): thresholds are
# processed by increasing height in the elimination tree of A + A^T,
# all thresholds of one height in the same round; a vertex newly reached in
# the round of height h is a fill iff its height exceeds h, else it joins the
# round's closure.  Test-side model in plain Python (its own etree from the
# definition parent(v) = min{u > v : u adjacent to the component of v in
# G(A+A^T) restricted to {0..v}}), checked against the oracle.

def etree_by_definition(rp, ci):
    n = rp.size - 1
    adj = [set() for _ in range(n)]
    for i in range(n):
        for j in ci[rp[i]:rp[i + 1]].tolist():
            if j != i:
                adj[i].add(j)
                adj[j].add(i)
    parent = [-1] * n
    for v in range(n):
        comp, stack = {v}, [v]          # component of v in G[{0..v}]
        while stack:
            x = stack.pop()
            for y in adj[x]:
                if y <= v and y not in comp:
                    comp.add(y)
                    stack.append(y)
        higher = [u for x in comp for u in adj[x] if u > v]
        parent[v] = min(higher) if higher else -1
    height = [0] * n
    for v in range(n):
        if parent[v] >= 0:
            height[parent[v]] = max(height[parent[v]], height[v] + 1)
    return parent, height


def height_order_source(rp, ci, src, height, rounds=None):
    n = rp.size - 1
    reached = {src}
    instruct = set()
    bucket = {}
    for w in ci[rp[src]:rp[src + 1]].tolist():
        if w == src:
            continue
        instruct.add(w)
        if w < src:
            reached.add(w)
            bucket.setdefault(height[w], set()).add(w)
    nround = 0
    while bucket:
        h = min(bucket)
        frontier = sorted(bucket.pop(h))
        nround += 1
        while frontier:
            nxt = []
            for u in frontier:
                for w in ci[rp[u]:rp[u + 1]].tolist():
                    if w == src:
                        continue
                    if w > src:
                        instruct.add(w)
                        continue
                    if w in reached:
                        continue
                    reached.add(w)
                    assert height[w] != h        # neither ancestor nor descendant: impossible
                    if height[w] > h:            # an ancestor of its threshold: fill
                        assert height[w] > h
                        instruct.add(w)
                        bucket.setdefault(height[w], set()).add(w)
                    else:                        # a descendant: the round's closure
                        nxt.append(w)
            frontier = nxt
    if rounds is not None:
        rounds.append(nround)
    return sorted(instruct)


@pytest.mark.parametrize("seed", range(60))
def test_height_order_reaches_oracle(seed):
    rng = np.random.default_rng(seed)
    n = int(rng.integers(8, 80))
    rp, ci = gen.random_graph(n, float(rng.uniform(0.02, 0.25)), seed=9100 + seed)
    _, height = etree_by_definition(rp, ci)
    r = oracle.rows(rp, ci)
    for src in range(n):
        want = sorted(set(r["L_colidx"][r["L_rowptr"][src]:r["L_rowptr"][src + 1]].tolist())
                      | set(r["U_colidx"][r["U_rowptr"][src] + 1:r["U_rowptr"][src + 1]].tolist()))
        assert height_order_source(rp, ci, src, height) == want, src


@pytest.mark.parametrize("name,scale", [("C4", 20), ("C5", 7), ("C2", 8)])
def test_height_order_rounds_on_grid(name, scale):
    """On nested-dissection grids the top rows need fewer rounds in height
    order than their threshold counts |L(s,:)| (the chain of id order), with
    the same structure."""
    rp, ci = gen.config(name, scale)
    n = rp.size - 1
    _, height = etree_by_definition(rp, ci)
    r = oracle.rows(rp, ci, np.array([n - 1], np.int64))
    rounds = []
    got = height_order_source(rp, ci, n - 1, height, rounds)
    want = sorted(set(r["L_colidx"].tolist()) | set(r["U_colidx"][1:].tolist()))
    assert got == want
    nL = int(r["L_rowptr"][1])
    assert rounds[0] <= nL                 # every round takes at least one threshold
    if name == "C4":
        assert rounds[0] < nL / 2          # 2D ND: a bushy tree
