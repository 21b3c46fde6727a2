"""Generator checks: determinism, CSR invariants, the shapes BASELINE.json and
Table 1 ask for."""
import numpy as np
import pytest

import gen


def _check_csr(rp, ci):
    n = rp.size - 1
    assert rp.dtype == np.int64 and ci.dtype == np.int32
    assert rp[0] == 0 and rp[-1] == ci.size and np.all(np.diff(rp) >= 0)
    assert ci.size == 0 or (ci.min() >= 0 and ci.max() < n)
    rows = np.repeat(np.arange(n), np.diff(rp))
    assert np.all(ci != rows)                      # diagonal implicit
    same = rows[1:] == rows[:-1]
    assert np.all(ci[1:][same] > ci[:-1][same])    # strictly increasing


def test_deterministic():
    a = gen.config("C1")
    b = gen.config("C1")
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])


def test_nd_order_is_permutation_and_separator_last():
    k = 16
    new = gen.nd_order((k, k, k))
    assert np.array_equal(np.sort(new), np.arange(k ** 3))
    coords = np.stack(np.unravel_index(np.arange(k ** 3), (k, k, k)), axis=1)
    top = new >= k ** 3 - k * k        # the top separator is the middle plane
    assert np.all(coords[top, 0] == k // 2)


@pytest.mark.parametrize("name", ["C1", "C2", "C3"])
def test_config_shapes(name):
    rp, ci = gen.config(name)
    _check_csr(rp, ci)
    st = gen.csr_stats(rp, ci)
    if name == "C1":
        assert st["n"] == 1024 and abs(st["symmetry"] - 0.75) < 0.05
    if name == "C2":
        assert st["n"] == 64 ** 3 and abs(st["nnz_offdiag"] - 1548288 * 0.75) < 5000
    if name == "C3":   # BBMAT, Table 1
        assert st["n"] == 38744
        assert abs(st["nnz_with_diag"] - 1771722) / 1771722 < 0.01
        assert abs(st["symmetry"] - 0.53) < 0.02


@pytest.mark.slow
def test_config_shapes_large():
    rp, ci = gen.config("C4")
    _check_csr(rp, ci)
    st = gen.csr_stats(rp, ci)
    assert st["n"] == 1585478 and abs(st["nnz_with_diag"] - 7660826) / 7660826 < 0.01
    assert st["symmetry"] == 1.0


def test_small_shapes():
    for rp, ci in [gen.paper_example(), gen.random_graph(30, 0.1, 1),
                   gen.config("C4", 20), gen.config("C5", 6), gen.config("C3", 900)]:
        _check_csr(rp, ci)
