"""Pins for the CPU oracle (oracle/), independent of the oracle's own code.

Each pin is something the paper or the mathematics fixes, chosen so that a
plausible mistake in oracle.c (a dropped neighbour, a wrong comparison
direction, L/U swapped, the diagonal mis-counted, a wrong supernode rule)
fails at least one of them:

* dense 0/1 Gaussian elimination without pivoting
* per-pair restricted-path brute force of Theorem thm:fill
* the worked example
* closed form for the 2D k x k 5-point grid in natural order
* elimination-tree row structure for symmetric patterns
* special cases (diagonal, triangular, dense, tridiagonal, star, arrowhead)
* invariants: A in L+U, closure under elimination, monotonicity
* supernodes: the paper's two-phase algorithm written
  independently, Def. def:T3 re-check and maximality.
"""
import json
import os

import numpy as np
import pytest

import gen
import oracle

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "paper_example.json")


# ---------------------------------------------------------------- helpers ---

def dense_pattern(rowptr, colidx):
    n = rowptr.size - 1
    M = np.zeros((n, n), dtype=bool)
    rows = np.repeat(np.arange(n), np.diff(rowptr))
    M[rows, colidx] = True
    np.fill_diagonal(M, True)
    return M


def dense_ge(rowptr, colidx):
    """0/1 Gaussian elimination: for each pivot k, every row i > k
    with a nonzero in column k receives row k's pattern right of k."""
    M = dense_pattern(rowptr, colidx)
    n = M.shape[0]
    for k in range(n):
        rows = np.nonzero(M[k + 1:, k])[0] + k + 1
        if rows.size:
            M[rows, k + 1:] |= M[k, k + 1:]
    return M


def brute_fill_path(rowptr, colidx):
    """Theorem thm:fill written out: (i,j) in L+U iff A(i,j) != 0 or j is
    reachable from i through intermediates all < min(i,j)."""
    n = rowptr.size - 1
    M = np.zeros((n, n), dtype=bool)
    for i in range(n):
        M[i, i] = True
        for j in range(n):
            if j == i:
                continue
            lim = min(i, j)
            seen = {i}
            stack = [i]
            found = False
            while stack and not found:
                u = stack.pop()
                for w in colidx[rowptr[u]:rowptr[u + 1]]:
                    w = int(w)
                    if w == j:
                        found = True
                        break
                    if w < lim and w not in seen:
                        seen.add(w)
                        stack.append(w)
            M[i, j] = found
    return M


def oracle_dense(rowptr, colidx):
    n = rowptr.size - 1
    r = oracle.rows(rowptr, colidx, nthreads=2)
    M = np.zeros((n, n), dtype=bool)
    for i in range(n):
        Li = r["L_colidx"][r["L_rowptr"][i]:r["L_rowptr"][i + 1]]
        Ui = r["U_colidx"][r["U_rowptr"][i]:r["U_rowptr"][i + 1]]
        assert np.all(Li < i) and np.all(np.diff(Li) > 0)
        assert Ui.size >= 1 and Ui[0] == i and np.all(np.diff(Ui) > 0)
        M[i, Li] = True
        M[i, Ui] = True
    return M, r


def row_sets(r, i):
    L = r["L_colidx"][r["L_rowptr"][i]:r["L_rowptr"][i + 1]]
    U = r["U_colidx"][r["U_rowptr"][i]:r["U_rowptr"][i + 1]]
    return L, U


# --------------------------------------------------- brute-force pins -------

@pytest.mark.parametrize("seed", range(300))
def test_oracle_equals_dense_ge_random(seed):
    rng = np.random.default_rng(seed)
    n = int(rng.integers(8, 65))
    dens = float(rng.uniform(0.02, 0.20))
    rp, ci = gen.random_graph(n, dens, seed=1000 + seed)
    M, _ = oracle_dense(rp, ci)
    assert np.array_equal(M, dense_ge(rp, ci))


@pytest.mark.parametrize("seed", range(40))
def test_oracle_equals_fill_path_brute_force(seed):
    rng = np.random.default_rng(50_000 + seed)
    n = int(rng.integers(6, 22))
    rp, ci = gen.random_graph(n, float(rng.uniform(0.05, 0.3)), seed=2000 + seed)
    M, _ = oracle_dense(rp, ci)
    assert np.array_equal(M, brute_fill_path(rp, ci))
    assert np.array_equal(M, dense_ge(rp, ci))


@pytest.mark.parametrize("name,scale", [("C1", None), ("C2", 10), ("C3", 1500), ("C4", 24), ("C5", 8)])
def test_oracle_equals_dense_ge_config_shapes(name, scale):
    rp, ci = gen.config(name, scale)
    M, _ = oracle_dense(rp, ci)
    assert np.array_equal(M, dense_ge(rp, ci))


def test_oracle_ignores_input_diagonal():
    rp, ci = gen.random_graph(40, 0.1, seed=7)
    n = rp.size - 1
    rows = np.repeat(np.arange(n), np.diff(rp))
    rp2, ci2 = gen.csr_from_edges(n, rows, ci)  # same graph
    # add explicit diagonal entries by hand (csr_from_edges drops them)
    src = np.concatenate([rows, np.arange(n)])
    dst = np.concatenate([ci, np.arange(n)])
    key = np.unique(src * n + dst)
    cnt = np.bincount(key // n, minlength=n)
    rp3 = np.concatenate([[0], np.cumsum(cnt)]).astype(np.int64)
    ci3 = (key % n).astype(np.int32)
    a = oracle.rows(rp2, ci2)
    b = oracle.rows(rp3, ci3)
    for k in ("L_rowptr", "L_colidx", "U_rowptr", "U_colidx"):
        assert np.array_equal(a[k], b[k])


# ----------------------------------------------------- worked example -------

def test_paper_example_facts():
    g = json.load(open(GOLDEN))
    rp, ci = gen.paper_example()
    # the fixture's edge list is the generator's graph
    for u in range(g["n"]):
        want = sorted(g["edges"].get(str(u), []))
        assert list(ci[rp[u]:rp[u + 1]]) == want
    r = oracle.symbolic(rp, ci, chunk_size=128)
    L8, U8 = row_sets(r, 8)
    A8 = set(ci[rp[8]:rp[9]].tolist())
    fills8 = sorted((set(L8.tolist()) | set(U8.tolist())) - A8 - {8})
    assert fills8 == g["row8_fills"]["value"]
    L1, U1 = row_sets(r, 1)
    assert 5 in U1.tolist() and 5 not in ci[rp[1]:rp[2]].tolist()       # fill (1,5)
    assert U1.size == g["nnzU_row1"]["value"]
    assert row_sets(r, 0)[1].size == g["nnzU_row0"]["value"]
    assert (0 in L1.tolist()) == g["L_1_0"]["value"]
    assert (0 in row_sets(r, 2)[0].tolist()) == g["L_2_0"]["value"]
    # supernodes over rows 0..3: blocks {0,1},{2},{3}
    blocks = g["blocks_rows0to3"]["value"]
    sn = r["sn_start"].tolist()
    assert sn[:3] == [b[0] for b in blocks]
    assert sn[3] == 4  # row 3 is alone: the next block starts at 4


# ------------------------------------------------------- closed forms -------

@pytest.mark.parametrize("k", list(range(1, 13)) + [32])
def test_grid2d_natural_closed_form(k):
    """k x k 5-point grid, natural order, no dropout: the band of width k
    fills completely: nnz(L) = nnz(U) - n = (k-1)(k^2+1), fill = 2(k-1)^3."""
    rp, ci = gen.grid2d(k, p=0.0, seed=0, order="natural")
    r = oracle.symbolic(rp, ci)
    n = k * k
    assert r["nnz_L"] == (k - 1) * (k * k + 1)
    assert r["nnz_U"] - n == (k - 1) * (k * k + 1)
    assert r["fill_count"] == 2 * (k - 1) ** 3


# ------------------------------------------- symmetric: elimination tree ----

def etree(rowptr, colidx):
    """Liu's elimination tree with path compression (symmetric pattern)."""
    n = rowptr.size - 1
    parent = -np.ones(n, dtype=np.int64)
    anc = -np.ones(n, dtype=np.int64)
    for i in range(n):
        for k in colidx[rowptr[i]:rowptr[i + 1]]:
            k = int(k)
            if k >= i:
                continue
            r = k
            while anc[r] != -1 and anc[r] != i:
                t = anc[r]
                anc[r] = i
                r = t
            if anc[r] == -1:
                anc[r] = i
                parent[r] = i
    return parent


def cholesky_rows(rowptr, colidx):
    """Row structure of the Cholesky factor from the etree (row subtrees,
    P:264): L(i,:) = union over k in A(i, <i) of the etree path k -> i."""
    n = rowptr.size - 1
    parent = etree(rowptr, colidx)
    mark = -np.ones(n, dtype=np.int64)
    rows = []
    for i in range(n):
        mark[i] = i
        s = []
        for k in colidx[rowptr[i]:rowptr[i + 1]]:
            k = int(k)
            if k >= i:
                continue
            while mark[k] != i:
                s.append(k)
                mark[k] = i
                k = int(parent[k])
        rows.append(sorted(s))
    return rows


def symmetrize(rowptr, colidx):
    n = rowptr.size - 1
    rows = np.repeat(np.arange(n), np.diff(rowptr))
    return gen.csr_from_edges(n, np.concatenate([rows, ci64(colidx)]), np.concatenate([ci64(colidx), rows]))


def ci64(c):
    return np.asarray(c, dtype=np.int64)


@pytest.mark.parametrize("case", ["rand", "grid3d_nd", "grid2d_nd", "circuit", "C4shape"])
def test_symmetric_matches_cholesky_etree(case):
    if case == "rand":
        rp, ci = symmetrize(*gen.random_graph(120, 0.03, seed=11))
    elif case == "grid3d_nd":
        rp, ci = gen.grid3d(9, p=0.0, seed=0, order="nd")
    elif case == "grid2d_nd":
        rp, ci = gen.grid2d(30, p=0.0, seed=0, order="nd")
    elif case == "circuit":
        rp, ci = gen.circuit_like(side=30, nhubs=6, hub_degree_sum=200, seed=9)
    else:
        rp, ci = gen.config("C4", 40)
    r = oracle.rows(rp, ci)
    chol = cholesky_rows(rp, ci)
    n = rp.size - 1
    Lt = [[] for _ in range(n)]
    for i in range(n):
        L, U = row_sets(r, i)
        assert L.tolist() == chol[i]
        for j in L.tolist():
            Lt[j].append(i)
    for j in range(n):          # U_strict = L^T for symmetric patterns
        assert row_sets(r, j)[1][1:].tolist() == Lt[j]


# ------------------------------------------------------ special cases -------

def _csr(n, edges):
    e = np.array(edges, dtype=np.int64).reshape(-1, 2)
    return gen.csr_from_edges(n, e[:, 0], e[:, 1])


def test_special_cases():
    n = 12
    # diagonal only: no fill, every row U = {i}
    r = oracle.symbolic(*_csr(n, []))
    assert r["fill_count"] == 0 and r["nnz_L"] == 0 and r["nnz_U"] == n
    # lower-triangular dense: no path climbs above the source -> no fill
    r = oracle.symbolic(*_csr(n, [(i, j) for i in range(n) for j in range(i)]))
    assert r["fill_count"] == 0
    # dense: nothing to fill
    r = oracle.symbolic(*_csr(n, [(i, j) for i in range(n) for j in range(n) if i != j]))
    assert r["fill_count"] == 0 and r["nnz_L"] == n * (n - 1) // 2
    # tridiagonal: no fill
    r = oracle.symbolic(*_csr(n, [(i, i + 1) for i in range(n - 1)] + [(i + 1, i) for i in range(n - 1)]))
    assert r["fill_count"] == 0
    # star centred at vertex 0 (both directions): complete fill
    r = oracle.symbolic(*_csr(n, [(0, v) for v in range(1, n)] + [(v, 0) for v in range(1, n)]))
    assert r["nnz_L"] + r["nnz_U"] == n * n
    # arrowhead with the hub last: no fill
    h = n - 1
    r = oracle.symbolic(*_csr(n, [(h, v) for v in range(h)] + [(v, h) for v in range(h)]))
    assert r["fill_count"] == 0


# ---------------------------------------------------------- invariants ------

@pytest.mark.parametrize("seed", range(20))
def test_invariants_containment_closure_monotone(seed):
    rng = np.random.default_rng(900 + seed)
    n = int(rng.integers(20, 80))
    rp, ci = gen.random_graph(n, float(rng.uniform(0.02, 0.1)), seed=3000 + seed)
    M, r = oracle_dense(rp, ci)
    A = dense_pattern(rp, ci)
    assert np.all(M[A])                             # pattern(A) in pattern(L+U)
    # closure (perfect elimination): (i,k) in L and (k,j) in U, j != i -> (i,j)
    for i in range(n):
        for k in np.nonzero(M[i, :i])[0]:
            js = np.nonzero(M[k, k + 1:])[0] + k + 1
            js = js[js != i]
            assert np.all(M[i, js])
    # monotone: adding an edge never removes an entry
    u, v = int(rng.integers(0, n)), int(rng.integers(0, n))
    rows = np.repeat(np.arange(n), np.diff(rp))
    rp2, ci2 = gen.csr_from_edges(n, np.append(rows, u), np.append(ci64(ci), v))
    M2, _ = oracle_dense(rp2, ci2)
    assert np.all(M2[M])


# ---------------------------------------------------------- supernodes ------

def two_phase_supernodes(nnzU, Lsets, chunk, row_begin=0):
    """The paper's two-phase SIMT design per chunk:
    Phase I bit[s] = nnzU(s) == nnzU(s-1) - 1 (chunk starts get 0); leaders =
    rows with bit 0.  Phase II: every leader grows through following rows
    while bit[s] and L(s, leader) != 0; rows that are not absorbed become
    leaders; repeat until no supernode grows."""
    m = len(nnzU)
    starts = []
    c0 = 0
    while c0 < m:
        s_abs = row_begin + c0
        c1 = min(m, c0 + (chunk - (s_abs % chunk)))
        bits = [0] + [int(nnzU[s] == nnzU[s - 1] - 1) for s in range(c0 + 1, c1)]
        leaders = [c0 + i for i, b in enumerate(bits) if b == 0]
        owner = {}
        frontier = list(leaders)
        while frontier:
            new = []
            for r in frontier:
                s = r + 1
                while s < c1 and bits[s - c0] and s not in owner and s not in leaders \
                        and (row_begin + r) in Lsets[s]:
                    owner[s] = r
                    s += 1
                if s < c1 and s not in owner and s not in leaders:
                    new.append(s)        # rejected row: becomes a leader
                    leaders.append(s)
            frontier = new
        starts += sorted(row_begin + x for x in leaders)
        c0 = c1
    return starts + [row_begin + m]


@pytest.mark.parametrize("seed", range(60))
def test_supernodes_two_phase_and_def1(seed):
    rng = np.random.default_rng(7000 + seed)
    n = int(rng.integers(10, 90))
    if seed % 3 == 0:
        rp, ci = gen.grid3d(4, p=0.25, seed=seed, order="nd")
    else:
        rp, ci = gen.random_graph(n, float(rng.uniform(0.03, 0.25)), seed=5000 + seed)
    n = rp.size - 1
    for chunk in (1, 2, 3, 4, 7, 128):
        r = oracle.symbolic(rp, ci, chunk_size=chunk)
        nnzU = np.diff(r["U_rowptr"]).tolist()
        Ls = [set(row_sets(r, i)[0].tolist()) for i in range(n)]
        sn = r["sn_start"].tolist()
        assert sn == two_phase_supernodes(nnzU, Ls, chunk)
        # Def. def:T3 re-check on every interior row + maximality of leaders
        for b in range(len(sn) - 1):
            lead = sn[b]
            assert sn[b + 1] - lead <= chunk
            for s in range(lead + 1, sn[b + 1]):
                assert nnzU[s] == nnzU[s - 1] - 1 and lead in Ls[s]
            if b > 0 and lead % chunk != 0:
                prev = sn[b - 1]
                assert not (nnzU[lead] == nnzU[lead - 1] - 1 and prev in Ls[lead])
        if chunk == 1:
            assert sn == list(range(n + 1))


def test_supernodes_row_range_subset():
    rp, ci = gen.grid3d(5, p=0.25, seed=4, order="nd")
    full = oracle.symbolic(rp, ci, chunk_size=8)
    part = oracle.symbolic(rp, ci, chunk_size=8, row_begin=40, row_end=100)
    # a chunk-aligned range reproduces the full partition restricted to it
    inside = [s for s in full["sn_start"].tolist() if 40 <= s < 100] + [100]
    assert part["sn_start"].tolist() == inside


# ------------------------------------- the second oracle (Gilbert-Peierls) --
# oracle.gp (oracle/gp.c): column-by-column reach through the columns of L
# computed so far.  Independent of oracle.c (fill2 per row); both
# are pinned to dense 0/1 Gaussian elimination here and to each other at mid
# scale.

def gp_dense(rowptr, colidx):
    n = rowptr.size - 1
    r = oracle.gp(rowptr, colidx)
    M = np.zeros((n, n), dtype=bool)
    for i in range(n):
        Li = r["L_colidx"][r["L_rowptr"][i]:r["L_rowptr"][i + 1]]
        Ui = r["U_colidx"][r["U_rowptr"][i]:r["U_rowptr"][i + 1]]
        assert np.all(Li < i) and np.all(np.diff(Li) > 0)
        assert Ui.size >= 1 and Ui[0] == i and np.all(np.diff(Ui) > 0)
        M[i, Li] = True
        M[i, Ui] = True
    return M


@pytest.mark.parametrize("seed", range(100))
def test_gp_equals_dense_ge_random(seed):
    rng = np.random.default_rng(70_000 + seed)
    n = int(rng.integers(1, 65))
    rp, ci = gen.random_graph(n, float(rng.uniform(0.02, 0.25)), seed=3000 + seed)
    assert np.array_equal(gp_dense(rp, ci), dense_ge(rp, ci))


def test_gp_paper_example():
    """The worked example's row 8: L(8,:) = {1,2,3,4,5,7},
    U(8,:) = {8,9}; fill (1,5)."""
    rp, ci = gen.paper_example()
    r = oracle.gp(rp, ci)
    L8 = r["L_colidx"][r["L_rowptr"][8]:r["L_rowptr"][9]].tolist()
    U8 = r["U_colidx"][r["U_rowptr"][8]:r["U_rowptr"][9]].tolist()
    assert L8 == [1, 2, 3, 4, 5, 7] and U8 == [8, 9]
    assert 5 in r["U_colidx"][r["U_rowptr"][1]:r["U_rowptr"][2]].tolist()


@pytest.mark.parametrize("name,scale", [("C1", None), ("C2", 16), ("C3", 4000), ("C4", 80),
                                        ("C5", 20)])
def test_gp_equals_fill2_mid_scale(name, scale):
    """The two oracles agree element by element at mid scale (n up to 8k)."""
    rp, ci = gen.config(name, scale)
    a = oracle.gp(rp, ci)
    b = oracle.rows(rp, ci)
    for k in ("L_rowptr", "L_colidx", "U_rowptr", "U_colidx"):
        assert np.array_equal(a[k], b[k]), k


# ------------------------------------ cap-only supernodes (§8(f) NEXT-3) ----
# chunk_size read only as the maximum supernode size, no forced
# breaks at its multiples.

def _diag_then_dense(p, m):
    """p diagonal-only rows, then an m x m dense block: rows p..p+m-1 hold
    every column of the block."""
    n = p + m
    rows, cols = [], []
    for i in range(p, n):
        for j in range(p, n):
            if i != j:
                rows.append(i)
                cols.append(j)
    return gen.csr_from_edges(n, np.array(rows, np.int64), np.array(cols, np.int64))


@pytest.mark.parametrize("p,m,cap", [(5, 40, 8), (3, 17, 4), (0, 30, 7), (6, 10, 128), (1, 9, 1)])
def test_cap_only_closed_form(p, m, cap):
    """Diagonal prefix + dense block (no fill): the prefix rows are singletons
    (nnzU = 1 each), the block's rows satisfy Def. def:T3 against any earlier
    block row (nnzU drops by one, L dense), so the cap-only blocks start at
    p, p + cap, p + 2 cap, ...; the forced-break partition instead breaks at
    the multiples of cap."""
    rp, ci = _diag_then_dense(p, m)
    n = p + m
    r = oracle.symbolic(rp, ci, chunk_size=cap, cap_only=True)
    assert r["fill_count"] == 0
    want = list(range(p)) + list(range(p, n, cap)) + [n]
    assert r["sn_start"].tolist() == want
    f = oracle.symbolic(rp, ci, chunk_size=cap)["sn_start"].tolist()
    want_f = sorted(set(range(p)) | {p} | {k for k in range(p, n) if k % cap == 0}) + [n]
    assert f == want_f


@pytest.mark.parametrize("seed", range(40))
def test_cap_only_def1_and_maximality(seed):
    """Every cap-only block satisfies Def. def:T3 and the cap; every leader
    after the first either follows a full block or fails (i) or (ii) against
    the previous leader (the greedy scan never splits a joinable row); with a
    cap of at least n both partitions are the uncapped greedy scan."""
    rng = np.random.default_rng(9100 + seed)
    if seed % 3 == 0:
        rp, ci = gen.grid3d(4, p=0.25, seed=seed, order="nd")
    else:
        rp, ci = gen.random_graph(int(rng.integers(10, 90)), float(rng.uniform(0.03, 0.3)),
                                  seed=9300 + seed)
    n = rp.size - 1
    for cap in (1, 2, 3, 5, 128):
        r = oracle.symbolic(rp, ci, chunk_size=cap, cap_only=True)
        nnzU = np.diff(r["U_rowptr"]).tolist()
        Ls = [set(row_sets(r, i)[0].tolist()) for i in range(n)]
        sn = r["sn_start"].tolist()
        assert sn[0] == 0 and sn[-1] == n and all(a < b for a, b in zip(sn, sn[1:]))
        for b in range(len(sn) - 1):
            lead = sn[b]
            assert sn[b + 1] - lead <= cap
            for s in range(lead + 1, sn[b + 1]):
                assert nnzU[s] == nnzU[s - 1] - 1 and lead in Ls[s]
            if b > 0 and lead - sn[b - 1] < cap:
                prev = sn[b - 1]
                assert not (nnzU[lead] == nnzU[lead - 1] - 1 and prev in Ls[lead])
        if cap == 1:
            assert sn == list(range(n + 1))
    big = oracle.symbolic(rp, ci, chunk_size=n + 1, cap_only=True)["sn_start"]
    assert np.array_equal(big, oracle.symbolic(rp, ci, chunk_size=n + 1)["sn_start"])



# ------------------- third comparator: etree row subtrees (§8(f) NEXT-4) ----
# oracle.etree_rows (oracle/etree.c): symmetric patterns only.

@pytest.mark.parametrize("seed", range(40))
def test_etree_rows_equals_dense_ge(seed):
    rng = np.random.default_rng(81_000 + seed)
    n = int(rng.integers(1, 70))
    rp, ci = symmetrize(*gen.random_graph(n, float(rng.uniform(0.01, 0.2)), seed=82_000 + seed))
    r = oracle.etree_rows(rp, ci)
    M = np.zeros((n, n), dtype=bool)
    for i in range(n):
        M[i, r["L_colidx"][r["L_rowptr"][i]:r["L_rowptr"][i + 1]]] = True
        M[i, r["U_colidx"][r["U_rowptr"][i]:r["U_rowptr"][i + 1]]] = True
    assert np.array_equal(M, dense_ge(rp, ci))


@pytest.mark.parametrize("k", [1, 2, 5, 12, 32])
def test_etree_rows_grid_closed_form(k):
    """2D k x k 5-point grid, natural order, no dropout: nnz(L) = (k-1)(k^2+1)."""
    rp, ci = gen.grid2d(k, p=0.0, seed=0, order="natural")
    r = oracle.etree_rows(rp, ci)
    assert int(r["L_rowptr"][-1]) == (k - 1) * (k * k + 1)
    assert int(r["U_rowptr"][-1]) - k * k == (k - 1) * (k * k + 1)


def test_etree_rows_rejects_nonsymmetric():
    rp, ci = gen.config("C1")  # p = 0.25 dropout per direction
    with pytest.raises(ValueError):
        oracle.etree_rows(rp, ci)


@pytest.mark.parametrize("name,scale", [("C4", 120), ("C4", None)])
def test_etree_rows_equal_fill2_symmetric_configs(name, scale):
    """C4 is structurally symmetric (G3_circuit is): the etree comparator and
    fill2 agree element by element (full size: 1.6M rows, a few seconds)."""
    rp, ci = gen.config(name, scale)
    a = oracle.etree_rows(rp, ci)
    b = oracle.rows(rp, ci)
    for key in ("L_rowptr", "L_colidx", "U_rowptr", "U_colidx"):
        assert np.array_equal(a[key], b[key]), key
