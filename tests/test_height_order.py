"""Plan step A2 host pass (gsofa_height_order, order.cu): the elimination
tree of A + A^T split over host threads (independent ND prefixes in
parallel, the rest in order), heights and (height, id) positions.

Pinned to the tree's definition: parent(k) = the smallest u > k
connected to k in G(A + A^T) restricted to {0..u} -- by brute force on small
patterns -- and, at larger sizes, the single-thread pass equals every thread
count.  No GPU needed (host computation through the C ABI)."""
import numpy as np
import pytest

import gen
import paper_2007_00840_b200 as g


def sym_adj(rowptr, colidx):
    n = rowptr.size - 1
    adj = [set() for _ in range(n)]
    for i in range(n):
        for j in colidx[rowptr[i]:rowptr[i + 1]]:
            j = int(j)
            if j != i:
                adj[i].add(j)
                adj[j].add(i)
    return adj


def parent_by_definition(rowptr, colidx):
    """parent(k) = min{u > k : k ~ u in G(A + A^T)[{0..u}]}.  The component
    C of k in G[{0..k}] only grows once a larger vertex touches it, so this
    is the smallest neighbour above k of C (brute force: one search per k)."""
    n = rowptr.size - 1
    adj = sym_adj(rowptr, colidx)
    parent = -np.ones(n, dtype=np.int64)
    for k in range(n):
        comp, stack, best = {k}, [k], n
        while stack:
            x = stack.pop()
            for w in adj[x]:
                if w > k:
                    best = min(best, w)
                elif w not in comp:
                    comp.add(w)
                    stack.append(w)
        if best < n:
            parent[k] = best
    return parent


def heights(parent):
    n = parent.size
    h = np.zeros(n, dtype=np.int64)
    for v in range(n):  # parents are larger
        if parent[v] >= 0:
            h[parent[v]] = max(h[parent[v]], h[v] + 1)
    return h


def check(rowptr, colidx, want_parent, threads, monkeypatch):
    monkeypatch.setenv("GSOFA_HOST_THREADS", str(threads))
    r = g.height_order(rowptr, colidx)
    n = rowptr.size - 1
    np.testing.assert_array_equal(r["parent"], want_parent)
    h = heights(want_parent)
    np.testing.assert_array_equal(r["hgt"], h)
    order = np.lexsort((np.arange(n), h))  # by (height, id)
    pos = np.empty(n, dtype=np.int64)
    pos[order] = np.arange(n)
    np.testing.assert_array_equal(r["pos"], pos)
    assert r["height"] == int(h.max())
    # last_row_chain: the union of tree paths from the last row's lower
    # neighbours (in A + A^T) up to it
    adj = sym_adj(rowptr, colidx)
    seen = set()
    for k in adj[n - 1]:
        while k != -1 and k < n - 1 and k not in seen:
            seen.add(k)
            k = int(want_parent[k])
    assert r["last_row_chain"] == len(seen)


SMALL = [
    ("paper", lambda: gen.paper_example()),
    ("grid2d_nat", lambda: gen.grid2d(9, seed=3)),
    ("grid3d_nd", lambda: gen.grid3d(6, seed=4)),
    ("grid3d_nat", lambda: gen.grid3d(5, seed=5, order="natural")),
    ("random", lambda: gen.random_graph(150, 0.02, 7)),
    ("random_sparse", lambda: gen.random_graph(200, 0.004, 8)),  # several components
    ("circuit", lambda: gen.circuit_like(side=12, nhubs=3, hub_degree_sum=60, symmetric=False)),
]


@pytest.mark.parametrize("threads", [1, 2, 3, 8])
@pytest.mark.parametrize("name,make", SMALL, ids=[s[0] for s in SMALL])
def test_height_order_definition(name, make, threads, monkeypatch):
    rp, ci = make()
    check(rp, ci, parent_by_definition(rp, ci), threads, monkeypatch)


MID = [
    ("C2_12", lambda: gen.config("C2", 12)),
    ("C4_60", lambda: gen.config("C4", 60)),
    ("C5_10", lambda: gen.config("C5", 10)),
    ("C3_s", lambda: gen.config("C3", 4)),
    ("grid3d_nat", lambda: gen.grid3d(14, seed=9, order="natural")),
    ("random", lambda: gen.random_graph(20000, 0.00015, 11)),
]


@pytest.mark.parametrize("name,make", MID, ids=[s[0] for s in MID])
def test_height_order_threads_agree(name, make, monkeypatch):
    """The split pass equals the sequential one (T = 1) for every thread
    count, on ND and non-ND patterns large enough to split."""
    rp, ci = make()
    monkeypatch.setenv("GSOFA_HOST_THREADS", "1")
    ref = g.height_order(rp, ci)
    for t in (2, 5, 16, 32):
        monkeypatch.setenv("GSOFA_HOST_THREADS", str(t))
        r = g.height_order(rp, ci)
        for k in ("parent", "hgt", "pos"):
            np.testing.assert_array_equal(r[k], ref[k], err_msg=f"{name} T={t} {k}")
        assert (r["height"], r["last_row_chain"]) == (ref["height"], ref["last_row_chain"])


def test_height_order_sequential_matches_definition_mid(monkeypatch):
    rp, ci = gen.config("C2", 7)
    check(rp, ci, parent_by_definition(rp, ci), 1, monkeypatch)


def test_height_order_errors():
    rp = np.array([0, 1, 2], dtype=np.int64)
    with pytest.raises(g.GsofaError):
        g.height_order(rp, np.array([1, 5], dtype=np.int32))  # column out of range
    with pytest.raises(g.GsofaError):
        g.height_order(np.array([0, 2, 1], dtype=np.int64), np.array([1, 0], dtype=np.int32))
    with pytest.raises(g.GsofaError):  # not strictly increasing
        g.height_order(np.array([0, 2, 2], dtype=np.int64), np.array([1, 1], dtype=np.int32))
