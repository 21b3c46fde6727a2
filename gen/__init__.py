"""Seeded synthetic input generators (shared by the oracle tests, the CUDA parity
tests, ``bench.py`` and ``smoke()``).

This module holds NONE of the method's arithmetic: it only builds sparsity
patterns (CSR of G(A)) with the shapes of the paper's workloads and of
``BASELINE.json:configs``.  Every generator is a pure function of its arguments
and an integer seed (numpy ``PCG64``), so the oracle side and the GPU side see
byte-identical inputs.

CSR convention: ``rowptr`` int64[n+1], ``colidx`` int32[nnz],
columns strictly increasing within a row, no diagonal entries (the diagonal is
implicit, "we do not represent the self edges").

Recipes (DESIGN.md "Input recipe" repeats them):

* C1  2D 5-point 32x32, natural order (id = 32*x + y), every directed
      off-diagonal edge dropped independently with p = 0.25, seed 1.
* C2  3D 7-point 64^3, geometric nested-dissection order, p = 0.25, seed 2.
* C3  BBMAT-shaped (Table 1: n = 38,744, nnz = 1,771,722, struct.
      symm. 0.53, nnz/n 45.7): banded random pattern, half-bandwidth b = 407 (calibrated with the oracle to fill/nnz ~ 18.3),
      each in-band (i, j) kept with prob q, mirrored with prob ``mirror``, plus
      one windowed scatter entry per row; natural (banded) order, seed 3.
* C4  G3_circuit-shaped: 1259^2 2D 5-point mesh (each undirected edge kept
      with prob 0.943), ND order, + 397 power-law (Zipf 2) hub vertices
      ordered last (ascending degree), hub edges to uniform mesh vertices,
      both directions; structurally symmetric; seed 4.
* C5  3D 7-point 128^3, ND order, p = 0.25, seed 5.

Nested dissection (geometric): recursive bisection of the box along its
longest axis (lowest axis index on ties), the middle plane is the separator
and is ordered after both halves; boxes of <= 8 vertices are leaves kept in
natural (lexicographic) order.
"""
from __future__ import annotations

import numpy as np

__all__ = [
    "csr_from_edges", "grid_edges", "nd_order", "grid2d", "grid3d",
    "bbmat_like", "circuit_like", "random_graph", "paper_example",
    "config", "CONFIGS", "csr_stats",
]


def _rng(seed: int) -> np.random.Generator:
    return np.random.Generator(np.random.PCG64(int(seed)))


def csr_from_edges(n: int, src: np.ndarray, dst: np.ndarray):
    """Build a CSR (rowptr int64, colidx int32) from directed edges; drops self
    edges and duplicates, sorts columns within each row."""
    src = np.asarray(src, dtype=np.int64)
    dst = np.asarray(dst, dtype=np.int64)
    keep = src != dst
    src, dst = src[keep], dst[keep]
    key = np.unique(src * np.int64(n) + dst)
    rows = key // n
    cols = (key % n).astype(np.int32)
    counts = np.bincount(rows, minlength=n).astype(np.int64)
    rowptr = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(counts, out=rowptr[1:])
    return rowptr, cols


def grid_edges(shape):
    """Undirected nearest-neighbour pairs (a, b), a < b, of a regular grid with
    lexicographic (natural) vertex ids."""
    shape = tuple(int(s) for s in shape)
    n = int(np.prod(shape))
    ids = np.arange(n, dtype=np.int64).reshape(shape)
    a_list, b_list = [], []
    for ax in range(len(shape)):
        if shape[ax] < 2:
            continue
        sl_a = [slice(None)] * len(shape)
        sl_b = [slice(None)] * len(shape)
        sl_a[ax] = slice(0, shape[ax] - 1)
        sl_b[ax] = slice(1, shape[ax])
        a_list.append(ids[tuple(sl_a)].ravel())
        b_list.append(ids[tuple(sl_b)].ravel())
    if not a_list:
        return np.zeros(0, np.int64), np.zeros(0, np.int64)
    return np.concatenate(a_list), np.concatenate(b_list)


def nd_order(shape, leaf: int = 8) -> np.ndarray:
    """Geometric nested-dissection order of a regular grid.

    Returns ``new_id`` (int64[n]) indexed by the natural (lexicographic) id.
    Vectorised level by level: each vertex carries its current box; at each
    level a non-leaf box is split at the middle plane of its longest axis into
    (left=0, right=1, separator=2); separator planes and leaf boxes terminate.
    Each vertex's base-4 digit string, left-aligned to a fixed length, sorted
    lexicographically with ties broken by natural id, is the ND order
    (separator after both halves, leaves in natural order).
    """
    shape = tuple(int(s) for s in shape)
    d = len(shape)
    n = int(np.prod(shape))
    depth = 31  # 2 bits per level -> 62-bit keys
    coords = np.stack(np.unravel_index(np.arange(n, dtype=np.int64), shape), axis=1)
    lo = np.zeros((n, d), dtype=np.int64)
    hi = np.tile(np.array(shape, dtype=np.int64) - 1, (n, 1))
    key = np.zeros(n, dtype=np.int64)
    active = np.ones(n, dtype=bool)
    for level in range(depth):
        idx = np.nonzero(active)[0]
        if idx.size == 0:
            break
        ext = hi[idx] - lo[idx] + 1
        small = np.prod(ext, axis=1) <= leaf
        active[idx[small]] = False
        idx, ext = idx[~small], ext[~small]
        if idx.size == 0:
            break
        ax = np.argmax(ext, axis=1)  # first max on ties
        mid = lo[idx, ax] + ext[np.arange(idx.size), ax] // 2
        x = coords[idx, ax]
        left, right = x < mid, x > mid
        sep = ~(left | right)
        shift = np.int64(2 * (depth - 1 - level))
        key[idx[right]] += np.int64(1) << shift
        key[idx[sep]] += np.int64(2) << shift
        active[idx[sep]] = False
        hi[idx[left], ax[left]] = mid[left] - 1
        lo[idx[right], ax[right]] = mid[right] + 1
    if active.any():
        raise RuntimeError("nd_order: grid too large for 31 levels")
    order = np.lexsort((np.arange(n, dtype=np.int64), key))  # old ids in new order
    new_id = np.empty(n, dtype=np.int64)
    new_id[order] = np.arange(n, dtype=np.int64)
    return new_id


def _relabel(n, a, b, new_id):
    if new_id is None:
        return a, b
    return new_id[a], new_id[b]


def _directed_dropout(a, b, p, rng):
    """Both directions of each undirected pair, each kept independently with
    probability 1 - p."""
    src = np.concatenate([a, b])
    dst = np.concatenate([b, a])
    if p > 0:
        keep = rng.random(src.size) >= p
        src, dst = src[keep], dst[keep]
    return src, dst


def grid2d(k: int, p: float = 0.25, seed: int = 1, order: str = "natural"):
    """2D 5-point k x k grid, id = k*x + y (natural) or ND."""
    rng = _rng(seed)
    a, b = grid_edges((k, k))
    src, dst = _directed_dropout(a, b, p, rng)
    new_id = nd_order((k, k)) if order == "nd" else None
    src, dst = _relabel(k * k, src, dst, new_id)
    return csr_from_edges(k * k, src, dst)


def grid3d(k: int, p: float = 0.25, seed: int = 2, order: str = "nd"):
    """3D 7-point k^3 grid, natural or ND order."""
    rng = _rng(seed)
    a, b = grid_edges((k, k, k))
    src, dst = _directed_dropout(a, b, p, rng)
    new_id = nd_order((k, k, k)) if order == "nd" else None
    src, dst = _relabel(k ** 3, src, dst, new_id)
    return csr_from_edges(k ** 3, src, dst)


def bbmat_like(n: int = 38744, b: int = 407, q: float = 0.0401,
               mirror: float = 0.36, scatter: int = 1, seed: int = 3):
    """BBMAT-shaped banded random pattern (Table 1).

    For every ordered pair (i, j) with 0 < |i - j| <= b the entry (i, j) is
    kept with probability q; a kept entry is mirrored to (j, i) with
    probability ``mirror``.  Each row also gets ``scatter`` entries at
    j = i + U[-2b, 2b] (clipped to [0, n)).  Natural (banded) order.
    """
    rng = _rng(seed)
    srcs, dsts = [], []
    offs = np.concatenate([np.arange(-b, 0), np.arange(1, b + 1)]).astype(np.int64)
    block = max(1, (1 << 22) // offs.size)
    for i0 in range(0, n, block):
        i1 = min(n, i0 + block)
        ii = np.repeat(np.arange(i0, i1, dtype=np.int64), offs.size)
        jj = ii + np.tile(offs, i1 - i0)
        ok = (jj >= 0) & (jj < n)
        ii, jj = ii[ok], jj[ok]
        keep = rng.random(ii.size) < q
        ii, jj = ii[keep], jj[keep]
        mir = rng.random(ii.size) < mirror
        srcs += [ii, jj[mir]]
        dsts += [jj, ii[mir]]
    for _ in range(scatter):
        ii = np.arange(n, dtype=np.int64)
        jj = np.clip(ii + rng.integers(-2 * b, 2 * b + 1, size=n), 0, n - 1)
        srcs.append(ii)
        dsts.append(jj)
    return csr_from_edges(n, np.concatenate(srcs), np.concatenate(dsts))


def circuit_like(side: int = 1259, nhubs: int = 397, keep: float = 0.943,
                 hub_degree_sum: int = 50000, seed: int = 4,
                 symmetric: bool = True):
    """G3_circuit-shaped graph: ND-ordered 2D mesh + power-law hubs last.

    Mesh: side x side 5-point grid, each undirected edge kept with prob
    ``keep`` (both directions), ND order.  Hubs: Zipf(2) degrees
    d_h = max(1, round(c / h^2)), c chosen so sum d_h ~ hub_degree_sum,
    ordered last by ascending degree; each hub edge goes to a uniformly
    random mesh vertex in both directions (``symmetric``) or each direction
    independently with prob 0.75 (nonsymmetric variant).
    """
    rng = _rng(seed)
    nm = side * side
    a, b = grid_edges((side, side))
    kept = rng.random(a.size) < keep
    a, b = a[kept], b[kept]
    new_id = nd_order((side, side))
    a, b = new_id[a], new_id[b]
    ranks = np.arange(1, nhubs + 1, dtype=np.float64)
    w = 1.0 / ranks ** 2
    deg = np.maximum(1, np.round(w * hub_degree_sum / w.sum())).astype(np.int64)
    deg = np.sort(deg)  # ascending degree -> hub ids nm .. nm+nhubs-1
    hub = np.repeat(np.arange(nm, nm + nhubs, dtype=np.int64), deg)
    tgt = rng.integers(0, nm, size=hub.size, dtype=np.int64)
    if symmetric:
        src = np.concatenate([a, b, hub, tgt])
        dst = np.concatenate([b, a, tgt, hub])
    else:
        s2 = np.concatenate([a, b, hub, tgt])
        d2 = np.concatenate([b, a, tgt, hub])
        k2 = rng.random(s2.size) >= 0.25
        src, dst = s2[k2], d2[k2]
    return csr_from_edges(nm + nhubs, src, dst)


def random_graph(n: int, density: float, seed: int):
    """Erdos-Renyi directed pattern: each off-diagonal (i, j) present with
    probability ``density``."""
    rng = _rng(seed)
    m = rng.random((n, n)) < density
    np.fill_diagonal(m, False)
    src, dst = np.nonzero(m)
    return csr_from_edges(n, src, dst)


def paper_example():
    """Reconstructed 10-vertex example of Fig. matrix_begin_end.

    Stated in the text: row 8 = {1, 2, 7, 9} off-diagonal; frontier
    neighbourhoods 1->{0}, 2->{3,5,7}, 7->{2,4}, 0->5, 3->4, 5->3;
    nonzero (1, 0).  Deduced: 0->1 (needed for nnz(U(0,:)) = 3 with
    the diagonal counted).  Out-edges of 4, 6, 9 are unknown (empty).
    """
    edges = {0: [1, 5], 1: [0], 2: [3, 5, 7], 3: [4], 5: [3], 7: [2, 4],
             8: [1, 2, 7, 9]}
    src = [i for i, js in edges.items() for _ in js]
    dst = [j for js in edges.values() for j in js]
    return csr_from_edges(10, np.array(src), np.array(dst))


CONFIGS = {
    "C1": dict(desc="2D 5-point 32x32, natural order, p=0.25 dropout, seed 1"),
    "C2": dict(desc="3D 7-point 64^3, ND order, p=0.25, seed 2"),
    "C3": dict(desc="BBMAT-shaped banded+scatter n=38,744, natural order, seed 3"),
    "C4": dict(desc="G3_circuit-shaped 1259^2 ND mesh + 397 hubs, n=1,585,478, seed 4"),
    "C5": dict(desc="3D 7-point 128^3, ND order, p=0.25, seed 5"),
}


def config(name: str, scale: int | None = None):
    """CSR of a BASELINE config (C1..C5).  ``scale`` shrinks the grid side
    (C2/C5: k, C4: mesh side, C3: n) for oracle-sized variants with the same
    recipe."""
    if name == "C1":
        return grid2d(scale or 32, 0.25, 1, "natural")
    if name == "C2":
        return grid3d(scale or 64, 0.25, 2, "nd")
    if name == "C3":
        return bbmat_like(n=scale or 38744, seed=3)
    if name == "C4":
        side = scale or 1259
        nh = 397 if scale is None else max(4, int(round(397 * side * side / 1259 ** 2)))
        hs = 50000 if scale is None else max(nh, int(50000 * side * side / 1259 ** 2))
        return circuit_like(side=side, nhubs=nh, hub_degree_sum=hs, seed=4)
    if name == "C5":
        return grid3d(scale or 128, 0.25, 5, "nd")
    raise KeyError(name)


def csr_stats(rowptr, colidx):
    """Shape statistics (Table 1 columns): n, nnz incl. diagonal,
    structural symmetry (fraction of off-diagonal (i,j) whose (j,i) exists)."""
    n = rowptr.size - 1
    rows = np.repeat(np.arange(n, dtype=np.int64), np.diff(rowptr))
    key = rows * n + colidx.astype(np.int64)
    tkey = colidx.astype(np.int64) * n + rows
    sym = np.isin(tkey, key).mean() if key.size else 1.0
    return dict(n=n, nnz_offdiag=int(colidx.size), nnz_with_diag=int(colidx.size + n),
                nnz_per_row=(colidx.size + n) / n, symmetry=float(sym))
