"""Matrix Market ingest (host IO): a sparse matrix file -> the pattern CSR the
library takes (rowptr int64[n+1], colidx int32[nnz], columns ascending,
diagonal dropped: it is implicit).  Values are ignored -- symbolic
factorization needs the pattern only.

Supported: ``%%MatrixMarket matrix coordinate {pattern|real|integer|complex}
{general|symmetric|skew-symmetric|hermitian}``, square.  Symmetric kinds store
one triangle; both directions are added.  The ordering is the file's; apply a
fill-reducing ordering with :func:`paper_2007_00840_b200.permute`.
"""
from __future__ import annotations

import gzip

import numpy as np


def read_matrix_market(path):
    opener = gzip.open if str(path).endswith(".gz") else open
    with opener(path, "rt") as f:
        header = f.readline().strip().split()
        if len(header) < 5 or header[0].lower() != "%%matrixmarket" or header[1].lower() != "matrix":
            raise ValueError(f"{path}: not a Matrix Market matrix file")
        fmt, field, sym = header[2].lower(), header[3].lower(), header[4].lower()
        if fmt != "coordinate":
            raise ValueError(f"{path}: only coordinate (sparse) files are supported, got {fmt}")
        if field not in ("pattern", "real", "integer", "complex", "double"):
            raise ValueError(f"{path}: unsupported field {field}")
        if sym not in ("general", "symmetric", "skew-symmetric", "hermitian"):
            raise ValueError(f"{path}: unsupported symmetry {sym}")
        line = f.readline()
        while line.startswith("%") or not line.strip():
            line = f.readline()
        nr, nc, nz = (int(x) for x in line.split()[:3])
        if nr != nc:
            raise ValueError(f"{path}: matrix is {nr} x {nc}, symbolic LU needs a square one")
        data = np.loadtxt(f, dtype=np.float64, ndmin=2, max_rows=nz, usecols=(0, 1)) if nz else \
            np.zeros((0, 2))
    if data.shape[0] != nz:
        raise ValueError(f"{path}: expected {nz} entries, read {data.shape[0]}")
    i = data[:, 0].astype(np.int64) - 1
    j = data[:, 1].astype(np.int64) - 1
    if nz and (i.min() < 0 or j.min() < 0 or i.max() >= nr or j.max() >= nr):
        raise ValueError(f"{path}: index out of range")
    if sym != "general":
        i, j = np.concatenate([i, j]), np.concatenate([j, i])
    keep = i != j
    key = np.unique(i[keep] * nr + j[keep])
    rows, cols = key // nr, (key % nr).astype(np.int32)
    rowptr = np.zeros(nr + 1, np.int64)
    np.cumsum(np.bincount(rows, minlength=nr), out=rowptr[1:])
    return rowptr, cols
