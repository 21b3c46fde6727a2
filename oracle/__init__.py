"""CPU oracle for gSoFa symbolic factorization -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import this package.  It
shares no code with the CUDA path (``paper_2007_00840_b200``).

``oracle.c`` implements, per row, the Rose-Tarjan fill2 traversal
 whose result is the fill-path structure of Theorem
thm:fill, and the greedy T3 supernode scan of Definition def:T3
 with forced breaks at multiples of chunk_size.

Pins (tests/test_oracle_pins.py, ``-m "not gpu"``): dense 0/1 Gaussian
elimination, per-pair restricted-path brute force (Theorem
thm:fill), the worked example,
the 2D-grid closed form, elimination-tree row counts for symmetric patterns
(P:264), special cases and invariants.  Parity pinned for every function.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_SRCS = [_SRC, os.path.join(_HERE, "gp.c"), os.path.join(_HERE, "etree.c")]
_LIB = os.path.join(_HERE, "liboracle.so")
_lib = None


def build(force: bool = False) -> str:
    """Compile oracle.c, gp.c and etree.c with gcc (plain C, -O2, pthreads)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < max(
            os.path.getmtime(f) for f in _SRCS):
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-fPIC", "-shared", "-pthread",
                               "-Wall", "-o", _LIB] + _SRCS)
    return _LIB


def _load():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(_LIB)
        P = ctypes.POINTER
        lib.oracle_rows.restype = ctypes.c_int
        lib.oracle_rows.argtypes = [
            ctypes.c_int64, P(ctypes.c_int64), P(ctypes.c_int32), P(ctypes.c_int64),
            ctypes.c_int64, ctypes.c_int,
            P(P(ctypes.c_int64)), P(P(ctypes.c_int32)), P(P(ctypes.c_int64)),
            P(P(ctypes.c_int32)), P(ctypes.c_int64)]
        lib.oracle_supernodes.restype = ctypes.c_int64
        lib.oracle_supernodes.argtypes = [
            ctypes.c_int64, ctypes.c_int64, P(ctypes.c_int64), P(ctypes.c_int32),
            P(ctypes.c_int64), ctypes.c_int64, P(ctypes.c_int32)]
        lib.oracle_supernodes_cap.restype = ctypes.c_int64
        lib.oracle_supernodes_cap.argtypes = lib.oracle_supernodes.argtypes
        lib.oracle_gp.restype = ctypes.c_int
        lib.oracle_gp.argtypes = [ctypes.c_int64, P(ctypes.c_int64), P(ctypes.c_int32),
                                  P(P(ctypes.c_int64)), P(P(ctypes.c_int32)),
                                  P(P(ctypes.c_int64)), P(P(ctypes.c_int32))]
        lib.oracle_etree_rows.restype = ctypes.c_int
        lib.oracle_etree_rows.argtypes = [ctypes.c_int64, P(ctypes.c_int64), P(ctypes.c_int32),
                                          ctypes.c_int, P(P(ctypes.c_int64)), P(P(ctypes.c_int32))]
        lib.oracle_free.restype = None
        lib.oracle_free.argtypes = [ctypes.c_void_p]
        _lib = lib
    return _lib


def _ptr(a, ct):
    return a.ctypes.data_as(ctypes.POINTER(ct))


def default_threads() -> int:
    return len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else os.cpu_count() or 1


def rows(rowptr, colidx, rows=None, nthreads: int | None = None):
    """struct(L(i,:)), struct(U(i,:)) for the requested rows (default: all).

    Returns dict(L_rowptr, L_colidx, U_rowptr, U_colidx, visits) with CSR over
    the requested rows in the given order; U includes the diagonal.
    """
    lib = _load()
    rowptr = np.ascontiguousarray(rowptr, dtype=np.int64)
    colidx = np.ascontiguousarray(colidx, dtype=np.int32)
    n = rowptr.size - 1
    if rows is None:
        rows = np.arange(n, dtype=np.int64)
    rows = np.ascontiguousarray(rows, dtype=np.int64)
    nthreads = nthreads or default_threads()
    P = ctypes.POINTER
    lp, li, up, ui = P(ctypes.c_int64)(), P(ctypes.c_int32)(), P(ctypes.c_int64)(), P(ctypes.c_int32)()
    visits = ctypes.c_int64(0)
    cidx = colidx if colidx.size else np.zeros(1, np.int32)
    rc = lib.oracle_rows(n, _ptr(rowptr, ctypes.c_int64), _ptr(cidx, ctypes.c_int32),
                         _ptr(rows, ctypes.c_int64) if rows.size else None, rows.size,
                         int(nthreads), ctypes.byref(lp), ctypes.byref(li), ctypes.byref(up),
                         ctypes.byref(ui), ctypes.byref(visits))
    if rc != 0:
        raise RuntimeError(f"oracle_rows failed rc={rc}")
    m = rows.size
    try:
        Lp = np.ctypeslib.as_array(lp, shape=(m + 1,)).copy()
        Up = np.ctypeslib.as_array(up, shape=(m + 1,)).copy()
        Li = np.ctypeslib.as_array(li, shape=(max(1, int(Lp[-1])),))[: int(Lp[-1])].copy()
        Ui = np.ctypeslib.as_array(ui, shape=(max(1, int(Up[-1])),))[: int(Up[-1])].copy()
    finally:
        for p in (lp, li, up, ui):
            lib.oracle_free(ctypes.cast(p, ctypes.c_void_p))
    return dict(L_rowptr=Lp, L_colidx=Li, U_rowptr=Up, U_colidx=Ui, visits=int(visits.value))


def supernodes(row_begin: int, L_rowptr, L_colidx, U_rowptr, chunk_size: int = 128,
               cap_only: bool = False):
    """Greedy T3 scan (Def. def:T3) over consecutive rows starting
    at ``row_begin``; returns sn_start (leading rows + sentinel).  Forced
    breaks at multiples of chunk_size, or with ``cap_only`` only a
    maximum supernode size of chunk_size rows."""
    lib = _load()
    Lp = np.ascontiguousarray(L_rowptr, dtype=np.int64)
    Li = np.ascontiguousarray(L_colidx, dtype=np.int32)
    Up = np.ascontiguousarray(U_rowptr, dtype=np.int64)
    m = Lp.size - 1
    out = np.zeros(m + 1, dtype=np.int32)
    Li_ = Li if Li.size else np.zeros(1, np.int32)
    fn = lib.oracle_supernodes_cap if cap_only else lib.oracle_supernodes
    ns = fn(int(row_begin), m, _ptr(Lp, ctypes.c_int64),
                               _ptr(Li_, ctypes.c_int32), _ptr(Up, ctypes.c_int64),
                               int(chunk_size), _ptr(out, ctypes.c_int32))
    if ns < 0:
        raise RuntimeError("oracle_supernodes: bad arguments")
    return out[: ns + 1].copy()


def symbolic(rowptr, colidx, chunk_size: int = 128, row_begin: int = 0,
             row_end: int | None = None, nthreads: int | None = None, cap_only: bool = False):
    """Full oracle result over rows [row_begin, row_end): L/U CSR, sn_start,
    nnz counts and fill count (nnz_offdiag(L+U) - nnz_offdiag(A))."""
    rowptr = np.asarray(rowptr, dtype=np.int64)
    colidx = np.asarray(colidx, dtype=np.int32)
    n = rowptr.size - 1
    row_end = n if row_end is None else row_end
    rr = np.arange(row_begin, row_end, dtype=np.int64)
    r = rows(rowptr, colidx, rr, nthreads)
    sn = supernodes(row_begin, r["L_rowptr"], r["L_colidx"], r["U_rowptr"], chunk_size, cap_only)
    rows_a = np.repeat(rr, np.diff(rowptr[row_begin:row_end + 1]))
    cols_a = colidx[rowptr[row_begin]:rowptr[row_end]]
    nnz_a_off = int(np.count_nonzero(cols_a != rows_a))
    nnz_L = int(r["L_rowptr"][-1])
    nnz_U = int(r["U_rowptr"][-1])
    fill = nnz_L + (nnz_U - rr.size) - nnz_a_off
    r.update(sn_start=sn, nsuper=int(sn.size - 1), nnz_L=nnz_L, nnz_U=nnz_U,
             nnz_A_offdiag=nnz_a_off, fill_count=int(fill), row_begin=row_begin,
             row_end=row_end)
    return r


def _cols_to_rows(cp, ri, n):
    """Column-compressed pattern -> row-compressed (rows' columns ascending)."""
    cols = np.repeat(np.arange(n, dtype=np.int64), np.diff(cp))
    order = np.lexsort((cols, ri))                      # by row, then column
    rows = ri[order].astype(np.int64)
    rp = np.zeros(n + 1, np.int64)
    np.add.at(rp, rows + 1, 1)
    return np.cumsum(rp), cols[order].astype(np.int32)


def gp(rowptr, colidx):
    """Second oracle: Gilbert-Peierls symbolic LU, column by
    column; returned in the same row form as :func:`symbolic` (L strictly
    lower, U with the diagonal first)."""
    lib = _load()
    rowptr = np.ascontiguousarray(rowptr, dtype=np.int64)
    colidx = np.ascontiguousarray(colidx, dtype=np.int32)
    n = rowptr.size - 1
    P = ctypes.POINTER
    lp, li, up, ui = P(ctypes.c_int64)(), P(ctypes.c_int32)(), P(ctypes.c_int64)(), P(ctypes.c_int32)()
    cidx = colidx if colidx.size else np.zeros(1, np.int32)
    rc = lib.oracle_gp(n, _ptr(rowptr, ctypes.c_int64), _ptr(cidx, ctypes.c_int32),
                       ctypes.byref(lp), ctypes.byref(li), ctypes.byref(up), ctypes.byref(ui))
    if rc != 0:
        raise RuntimeError(f"oracle_gp failed rc={rc}")
    try:
        Lp = np.ctypeslib.as_array(lp, shape=(n + 1,)).copy()
        Up = np.ctypeslib.as_array(up, shape=(n + 1,)).copy()
        Li = np.ctypeslib.as_array(li, shape=(max(1, int(Lp[-1])),))[: int(Lp[-1])].copy()
        Ui = np.ctypeslib.as_array(ui, shape=(max(1, int(Up[-1])),))[: int(Up[-1])].copy()
    finally:
        for q in (lp, li, up, ui):
            lib.oracle_free(ctypes.cast(q, ctypes.c_void_p))
    L_rowptr, L_colidx = _cols_to_rows(Lp, Li, n)
    U_rowptr, U_colidx = _cols_to_rows(Up, Ui, n)
    return dict(L_rowptr=L_rowptr, L_colidx=L_colidx, U_rowptr=U_rowptr, U_colidx=U_colidx)


def etree_rows(rowptr, colidx, nthreads: int | None = None):
    """Third comparator, symmetric patterns only: L by rows from the
    elimination tree's row subtrees (oracle/etree.c); U = L^T + diagonal.
    Returns dict(L_rowptr, L_colidx, U_rowptr, U_colidx); raises ValueError
    if the pattern is not structurally symmetric."""
    lib = _load()
    rowptr = np.ascontiguousarray(rowptr, dtype=np.int64)
    colidx = np.ascontiguousarray(colidx, dtype=np.int32)
    n = rowptr.size - 1
    P = ctypes.POINTER
    lp, li = P(ctypes.c_int64)(), P(ctypes.c_int32)()
    cidx = colidx if colidx.size else np.zeros(1, np.int32)
    rc = lib.oracle_etree_rows(n, _ptr(rowptr, ctypes.c_int64), _ptr(cidx, ctypes.c_int32),
                               int(nthreads or default_threads()), ctypes.byref(lp), ctypes.byref(li))
    if rc == -3:
        raise ValueError("pattern is not structurally symmetric")
    if rc != 0:
        raise RuntimeError(f"oracle_etree_rows failed rc={rc}")
    try:
        Lp = np.ctypeslib.as_array(lp, shape=(n + 1,)).copy()
        Li = np.ctypeslib.as_array(li, shape=(max(1, int(Lp[-1])),))[: int(Lp[-1])].copy()
    finally:
        for q in (lp, li):
            lib.oracle_free(ctypes.cast(q, ctypes.c_void_p))
    # U(i,:) = {i} + column i of L (symmetric pattern), ascending
    rows = np.repeat(np.arange(n, dtype=np.int64), np.diff(Lp))
    cols = Li.astype(np.int64)
    key_r = np.concatenate([cols, np.arange(n, dtype=np.int64)])
    key_c = np.concatenate([rows, np.arange(n, dtype=np.int64)])
    order = np.lexsort((key_c, key_r))
    Up = np.zeros(n + 1, np.int64)
    np.add.at(Up, key_r + 1, 1)
    return dict(L_rowptr=Lp, L_colidx=Li, U_rowptr=np.cumsum(Up),
                U_colidx=key_c[order].astype(np.int32))
