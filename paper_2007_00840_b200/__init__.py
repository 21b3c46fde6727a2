"""B200-native gSoFa symbolic LU factorization -- thin Python binding.

The product is the C-ABI shared library ``libgsofa.so`` (include/gsofa.h) built
from ``csrc/`` for sm_100a.  This module only marshals arguments (numpy arrays
or torch tensors in, numpy arrays / torch tensors out); every step of the
factorization runs in the library's CUDA kernels.  There is no CPU fallback:
if the library is missing or no GPU is usable, the calls raise.

Names follow include/gsofa.h: ``gsofa_symbolic`` -> :func:`symbolic`,
``gsofa_partition_rows`` -> :func:`partition_rows`, contexts ->
:class:`Context`.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

from .build import LIB_PATH, build  # noqa: F401

__all__ = ["Context", "Result", "Tail", "symbolic", "permute", "partition_rows", "height_order", "load", "GsofaError",
           "EXPORTED_SYMBOLS", "build", "LIB_PATH"]

EXPORTED_SYMBOLS = [
    "gsofa_default_opts", "gsofa_context_create", "gsofa_context_destroy",
    "gsofa_symbolic", "gsofa_result_copy", "gsofa_result_free",
    "gsofa_partition_rows", "gsofa_strerror", "gsofa_last_error_detail",
    "gsofa_version", "gsofa_supernode_stitch", "gsofa_result_l_csc", "gsofa_buffer_free",
    "gsofa_permute", "gsofa_result_supno", "gsofa_result_rowinfo", "gsofa_supernodes_gathered",
    "gsofa_height_order",
]

_I64, _I32 = ctypes.c_int64, ctypes.c_int32
_P = ctypes.POINTER


class Interleave(ctypes.Structure):
    """gsofa_interleave: units of unit_rows rows dealt round-robin to nparts
    parts; this call computes part `part`."""
    _fields_ = [("nparts", _I32), ("part", _I32), ("unit_rows", _I32), ("reserved", _I32)]


class Opts(ctypes.Structure):
    _fields_ = [("chunk_size", _I32), ("max_concurrent", _I32), ("mem_budget_bytes", _I64),
                ("fill_first", _I32), ("schedule", _I32), ("row_begin", _I64),
                ("row_end", _I64), ("device", _I32), ("outputs_on_device", _I32),
                ("stream", ctypes.c_void_p), ("checked", _I32),
                ("sn_cap_only", _I32), ("interleave", Interleave)]


class Stats(ctypes.Structure):
    _fields_ = [("edge_inspections", _I64), ("frontier_items", _I64), ("item_edges", _I64),
                ("rounds", _I64),
                ("thresholds", _I64), ("batches", _I64), ("max_batch", _I64), ("kernel_launches", _I64),
                ("ms_total", ctypes.c_double), ("ms_traverse", ctypes.c_double),
                ("ms_extract", ctypes.c_double), ("ms_supernode", ctypes.c_double),
                ("ms_transfer", ctypes.c_double), ("first_visits", _I64),
                ("source_expansions", _I64), ("frontier_spilled", _I64)]


class CResult(ctypes.Structure):
    _fields_ = [("n", _I64), ("row_begin", _I64), ("row_end", _I64),
                ("L_rowptr", _P(_I64)), ("L_colidx", _P(_I32)),
                ("U_rowptr", _P(_I64)), ("U_colidx", _P(_I32)),
                ("nsuper", _I64), ("sn_start", _P(_I32)),
                ("nnz_L", _I64), ("nnz_U", _I64), ("nnz_A_offdiag", _I64),
                ("fill_count", _I64), ("on_device", _I32), ("device", _I32),
                ("stats", Stats), ("schedule", _I32), ("reserved", _I32),
                ("rows", _I64), ("interleave", Interleave)]


class Tail(ctypes.Structure):
    """gsofa_tail: last row of a range, its nnz(U) and the leader of its block."""
    _fields_ = [("row", _I64), ("nnzU", _I64), ("leader", _I64)]

    def as_tuple(self):
        return (self.row, self.nnzU, self.leader)


class GsofaError(RuntimeError):
    def __init__(self, code, where, detail):
        super().__init__(f"{where} failed: code {code} ({detail})")
        self.code = code


_lib = None
SCHEDULES = {"threshold": 0, "fifo": 1, "auto": 2, "height": 3}
SCHEDULE_NAMES = {0: "threshold", 1: "fifo", 3: "height"}


def load():
    """Load libgsofa.so (never falls back to anything else)."""
    global _lib
    if _lib is not None:
        return _lib
    path = os.environ.get("GSOFA_LIB", LIB_PATH)  # dev: A/B a variant build
    if not os.path.exists(path):
        raise ImportError(f"{LIB_PATH} is missing: run __graft_entry__.build() "
                          "(nvcc -gencode arch=compute_100a,code=sm_100a)")
    lib = ctypes.CDLL(path)
    lib.gsofa_default_opts.argtypes = [_P(Opts)]
    lib.gsofa_context_create.argtypes = [_I32, _I64, _P(ctypes.c_void_p)]
    lib.gsofa_context_destroy.argtypes = [ctypes.c_void_p]
    lib.gsofa_context_destroy.restype = None
    lib.gsofa_symbolic.argtypes = [ctypes.c_void_p, _I64, ctypes.c_void_p, ctypes.c_void_p,
                                   _P(Opts), _P(_P(CResult))]
    lib.gsofa_result_copy.argtypes = [_P(CResult)] + [ctypes.c_void_p] * 5
    lib.gsofa_result_free.argtypes = [_P(CResult)]
    lib.gsofa_result_free.restype = None
    lib.gsofa_partition_rows.argtypes = [_I64, ctypes.c_void_p, ctypes.c_void_p, _I32, _I32,
                                         ctypes.c_void_p]
    lib.gsofa_height_order.argtypes = [_I64, ctypes.c_void_p, ctypes.c_void_p] + [ctypes.c_void_p] * 5
    lib.gsofa_supernode_stitch.argtypes = [_P(CResult), ctypes.c_void_p, ctypes.c_void_p]
    lib.gsofa_result_l_csc.argtypes = [_P(CResult), _I32, _P(_P(_I64)), _P(_P(_I32))]
    lib.gsofa_result_supno.argtypes = [_P(CResult), _I32, _P(_P(_I32))]
    lib.gsofa_buffer_free.argtypes = [ctypes.c_void_p, _I32]
    lib.gsofa_buffer_free.restype = None
    lib.gsofa_permute.argtypes = [_I64] + [ctypes.c_void_p] * 5
    lib.gsofa_result_rowinfo.argtypes = [_P(CResult), ctypes.c_void_p, ctypes.c_void_p]
    lib.gsofa_supernodes_gathered.argtypes = [_P(CResult), ctypes.c_void_p, ctypes.c_void_p, _I64]
    lib.gsofa_strerror.restype = ctypes.c_char_p
    lib.gsofa_strerror.argtypes = [ctypes.c_int]
    lib.gsofa_last_error_detail.restype = ctypes.c_char_p
    lib.gsofa_version.restype = ctypes.c_int
    _lib = lib
    return lib


def _check(rc, where):
    if rc != 0:
        lib = load()
        raise GsofaError(rc, where, f"{lib.gsofa_strerror(rc).decode()}: "
                                    f"{lib.gsofa_last_error_detail().decode()}")


def _ptr(a):
    """(pointer, is_device, keepalive) of a numpy array or torch tensor."""
    if isinstance(a, np.ndarray):
        if not a.flags["C_CONTIGUOUS"]:
            a = np.ascontiguousarray(a)
        return a.ctypes.data, False, a
    import torch
    if isinstance(a, torch.Tensor):
        a = a.contiguous()
        return a.data_ptr(), a.is_cuda, a
    raise TypeError(f"expected numpy array or torch tensor, got {type(a)}")


class Context:
    """Owns the device arena, stream and epoch counter (gsofa_context)."""

    def __init__(self, device: int = 0, mem_budget_bytes: int = 0):
        lib = load()
        h = ctypes.c_void_p()
        _check(lib.gsofa_context_create(int(device), int(mem_budget_bytes), ctypes.byref(h)),
               "gsofa_context_create")
        self._h = h
        self.device = device

    @property
    def handle(self):
        return self._h

    def close(self):
        if getattr(self, "_h", None):
            load().gsofa_context_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()


class Result:
    """A gsofa_result.  Host results expose numpy arrays; device results keep
    device memory until :meth:`free` and can be copied out with
    :meth:`to_numpy` or :meth:`to_torch`."""

    def __init__(self, cres_ptr):
        self._p = cres_ptr
        r = cres_ptr.contents
        self.n, self.row_begin, self.row_end = r.n, r.row_begin, r.row_end
        self.rows = r.rows
        iv = r.interleave
        self.interleave = (iv.nparts, iv.part, iv.unit_rows) if iv.nparts > 1 else None
        self.nnz_L, self.nnz_U, self.nsuper = r.nnz_L, r.nnz_U, r.nsuper
        self.nnz_A_offdiag, self.fill_count = r.nnz_A_offdiag, r.fill_count
        self.on_device = bool(r.on_device)
        self.device = r.device
        self.chunk_size = 128  # set by symbolic()
        self.schedule = SCHEDULE_NAMES.get(r.schedule, str(r.schedule))
        s = r.stats
        self.stats = {f: getattr(s, f) for f, _ in Stats._fields_}
        self._arrays = None

    def _sizes(self):
        return dict(L_rowptr=(self.rows + 1, np.int64), L_colidx=(self.nnz_L, np.int32),
                    U_rowptr=(self.rows + 1, np.int64), U_colidx=(self.nnz_U, np.int32),
                    sn_start=(self.nsuper + 1, np.int32))

    def to_numpy(self, copy: bool = True):
        """Arrays as numpy.  Host results with copy=False are zero-copy views
        of the library's (pinned) storage, valid until :meth:`free`."""
        if not self.on_device and not copy:
            r = self._p.contents
            views = {}
            for k, (sz, dt) in self._sizes().items():
                ptr = getattr(r, k)
                views[k] = (np.ctypeslib.as_array(ptr, shape=(max(sz, 1),))[:sz] if sz
                            else np.empty(0, dt))
            return views
        if self._arrays is None:
            out = {k: np.empty(sz, dt) for k, (sz, dt) in self._sizes().items()}
            self._copy(out)
            self._arrays = out
        return self._arrays

    def to_torch(self, device="cuda"):
        import torch
        tdt = {np.int64: torch.int64, np.int32: torch.int32}
        out = {k: torch.empty(sz, dtype=tdt[dt], device=device) for k, (sz, dt) in self._sizes().items()}
        self._copy(out)
        return out

    def _copy(self, out):
        ptrs = []
        for k in ("L_rowptr", "L_colidx", "U_rowptr", "U_colidx", "sn_start"):
            a = out[k]
            size = a.size if isinstance(a, np.ndarray) else a.numel()
            ptrs.append(_ptr(a)[0] if size else None)
        _check(load().gsofa_result_copy(self._p, *[ctypes.c_void_p(p) if p else None for p in ptrs]),
               "gsofa_result_copy")

    def stitch(self, prev=None) -> Tail:
        """gsofa_supernode_stitch: fix the head supernodes of this range from
        the predecessor's tail (a Tail, a (row, nnzU, leader) tuple, or None
        when row_begin starts a block); returns this range's tail."""
        if prev is not None and not isinstance(prev, Tail):
            prev = Tail(*[int(x) for x in prev])
        out = Tail()
        _check(load().gsofa_supernode_stitch(self._p, ctypes.byref(prev) if prev is not None else None,
                                             ctypes.byref(out)), "gsofa_supernode_stitch")
        self.nsuper = self._p.contents.nsuper
        self._arrays = None
        return out

    def rowinfo(self):
        """gsofa_result_rowinfo (device results): per local row nnz(U(s,:))
        (int32 tensor [rows]) and the candidate-leader L mask (int32 tensor
        [rows, W], W = ceil(chunk_size / 32), bit d: L(s, s - d) != 0)."""
        import torch
        lib = load()
        W = (self.chunk_size + 31) // 32
        nnzU = torch.empty(max(self.rows, 1), dtype=torch.int32, device=f"cuda:{self.device}")
        mask = torch.empty((max(self.rows, 1), W), dtype=torch.int32, device=f"cuda:{self.device}")
        _check(lib.gsofa_result_rowinfo(self._p, ctypes.c_void_p(nnzU.data_ptr()),
                                        ctypes.c_void_p(mask.data_ptr())), "gsofa_result_rowinfo")
        return nnzU[: self.rows], mask[: self.rows]

    def supernodes_gathered(self, nnzU_all, mask_all, stride: int):
        """gsofa_supernodes_gathered: this part's supernodes from every
        part's rowinfo, gathered part-major with `stride` rows per part
        (device tensors)."""
        _check(load().gsofa_supernodes_gathered(self._p, ctypes.c_void_p(nnzU_all.data_ptr()),
                                                ctypes.c_void_p(mask_all.data_ptr()), int(stride)),
               "gsofa_supernodes_gathered")
        self.nsuper = self._p.contents.nsuper
        self._arrays = None

    def l_csc(self):
        """gsofa_result_l_csc: L in compressed sparse column form, as numpy
        arrays col_ptr int64[n+1] (columns [0, n)) and row_idx int32[nnz_L]
        (rows ascending within each column)."""
        lib = load()
        cp, ri = _P(_I64)(), _P(_I32)()
        _check(lib.gsofa_result_l_csc(self._p, 0, ctypes.byref(cp), ctypes.byref(ri)),
               "gsofa_result_l_csc")
        try:
            col_ptr = np.ctypeslib.as_array(cp, shape=(self.n + 1,)).copy()
            row_idx = (np.ctypeslib.as_array(ri, shape=(self.nnz_L,)).copy() if self.nnz_L
                       else np.empty(0, np.int32))
        finally:
            lib.gsofa_buffer_free(ctypes.cast(cp, ctypes.c_void_p), 0)
            lib.gsofa_buffer_free(ctypes.cast(ri, ctypes.c_void_p), 0)
        return dict(col_ptr=col_ptr, row_idx=row_idx)

    def supno(self):
        """gsofa_result_supno: SuperLU's supno (xsup is sn_start): for each row
        of the range, the index of its supernode (numpy int32)."""
        lib = load()
        q = _P(_I32)()
        _check(lib.gsofa_result_supno(self._p, 0, ctypes.byref(q)), "gsofa_result_supno")
        try:
            return (np.ctypeslib.as_array(q, shape=(self.rows,)).copy() if self.rows
                    else np.empty(0, np.int32))
        finally:
            lib.gsofa_buffer_free(ctypes.cast(q, ctypes.c_void_p), 0)

    def __getitem__(self, k):
        return self.to_numpy()[k]

    def free(self):
        if self._p is not None:
            load().gsofa_result_free(self._p)
            self._p = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


def symbolic(rowptr, colidx, *, ctx: Context | None = None, chunk_size: int = 128,
             max_concurrent: int = 0, mem_budget_bytes: int = 0, fill_first: bool = False,
             row_begin: int = 0, row_end: int = -1, device: int = 0,
             outputs_on_device: bool = False, stream=None, schedule: str = "auto",
             checked: bool = False, sn_cap_only: bool = False, interleave=None) -> Result:
    """gsofa_symbolic: L/U patterns, supernodes and fill count of the pattern
    (rowptr int64[n+1], colidx int32[nnz]) for rows [row_begin, row_end).
    Inputs: numpy (host) or torch tensors (host or CUDA).  ``stream``: a
    torch.cuda.Stream or raw cudaStream_t integer.  ``schedule``:
    "auto" (default: FIFO for banded dense patterns, else threshold),
    "threshold" or "fifo" (the paper's all-frontiers order).  ``sn_cap_only``:
    chunk_size bounds the supernode size only (no forced breaks at its
    multiples).  ``interleave=(nparts, part, unit_rows)``:
    only this part's units of rows (gsofa_interleave)."""
    lib = load()
    rp, _, krp = _ptr(rowptr)
    ci, _, kci = _ptr(colidx)
    n = (krp.size if isinstance(krp, np.ndarray) else krp.numel()) - 1
    if isinstance(krp, np.ndarray):
        assert krp.dtype == np.int64 and kci.dtype == np.int32, "rowptr int64, colidx int32"
    o = Opts()
    lib.gsofa_default_opts(ctypes.byref(o))
    o.chunk_size, o.max_concurrent = int(chunk_size), int(max_concurrent)
    o.mem_budget_bytes, o.fill_first = int(mem_budget_bytes), int(bool(fill_first))
    o.row_begin, o.row_end, o.device = int(row_begin), int(row_end), int(device)
    o.outputs_on_device = int(bool(outputs_on_device))
    o.schedule = SCHEDULES[schedule]
    o.checked = int(bool(checked))
    o.sn_cap_only = int(bool(sn_cap_only))
    if interleave is not None:
        o.interleave.nparts, o.interleave.part, o.interleave.unit_rows = (int(x) for x in interleave)
    if stream is not None:
        o.stream = ctypes.c_void_p(stream if isinstance(stream, int) else stream.cuda_stream)
    if ci == 0:  # empty colidx: pass a valid dummy pointer
        dummy = np.zeros(1, np.int32)
        ci, kci = dummy.ctypes.data, dummy
    out = _P(CResult)()
    _check(lib.gsofa_symbolic(ctx.handle if ctx else None, n, ctypes.c_void_p(rp),
                              ctypes.c_void_p(ci), ctypes.byref(o), ctypes.byref(out)),
           "gsofa_symbolic")
    res = Result(out)
    res.chunk_size = int(chunk_size)
    return res


def partition_rows(rowptr, colidx, nparts: int, align: int = 1) -> np.ndarray:
    """gsofa_partition_rows: contiguous, align-multiple row ranges of equal
    estimated work (host computation); align=1: row-granular."""
    lib = load()
    rowptr = np.ascontiguousarray(rowptr, dtype=np.int64)
    colidx = np.ascontiguousarray(colidx, dtype=np.int32)
    if colidx.size == 0:
        colidx = np.zeros(1, np.int32)
    b = np.zeros(nparts + 1, dtype=np.int64)
    _check(lib.gsofa_partition_rows(rowptr.size - 1, rowptr.ctypes.data, colidx.ctypes.data,
                                    int(nparts), int(align), b.ctypes.data),
           "gsofa_partition_rows")
    return b


def height_order(rowptr, colidx) -> dict:
    """gsofa_height_order (host computation, plan step A2): elimination tree
    of A + A^T ("parent"), heights ("hgt"), (height, id) positions ("pos"),
    the tree "height" and the AUTO chain estimate "last_row_chain"."""
    lib = load()
    rowptr = np.ascontiguousarray(rowptr, dtype=np.int64)
    colidx = np.ascontiguousarray(colidx, dtype=np.int32)
    if colidx.size == 0:
        colidx = np.zeros(1, np.int32)
    n = rowptr.size - 1
    out = {k: np.zeros(n, np.int32) for k in ("parent", "hgt", "pos")}
    h, c = ctypes.c_int64(0), ctypes.c_int64(0)
    _check(lib.gsofa_height_order(n, rowptr.ctypes.data, colidx.ctypes.data, out["parent"].ctypes.data,
                                  out["hgt"].ctypes.data, out["pos"].ctypes.data, ctypes.byref(h),
                                  ctypes.byref(c)), "gsofa_height_order")
    out["height"], out["last_row_chain"] = h.value, c.value
    return out


def permute(rowptr, colidx, perm):
    """gsofa_permute: B = P A P^T (new vertex i = old vertex perm[i]) on the
    GPU; numpy in, numpy out (columns ascending per row)."""
    lib = load()
    rowptr = np.ascontiguousarray(rowptr, dtype=np.int64)
    colidx = np.ascontiguousarray(colidx, dtype=np.int32)
    perm = np.ascontiguousarray(perm, dtype=np.int32)
    n = rowptr.size - 1
    if perm.size != n:
        raise ValueError(f"perm has {perm.size} entries, expected n = {n}")
    out_rp = np.empty(n + 1, np.int64)
    out_ci = np.empty(max(colidx.size, 1), np.int32)
    ci = colidx if colidx.size else np.zeros(1, np.int32)
    _check(lib.gsofa_permute(n, rowptr.ctypes.data, ci.ctypes.data, perm.ctypes.data,
                             out_rp.ctypes.data, out_ci.ctypes.data), "gsofa_permute")
    return out_rp, out_ci[:colidx.size]
