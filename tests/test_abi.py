"""CPU-side checks of the C-ABI boundary (no compute calls without a GPU):
the library loads, exports every function include/gsofa.h declares, the
ctypes structures match the C layout, and the host-only partitioner works."""
import os
import re
import subprocess
import tempfile

import numpy as np
import pytest

import gen

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "gsofa.h")


@pytest.fixture(scope="module")
def g():
    import paper_2007_00840_b200 as mod
    mod.build()
    return mod


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(gsofa_[a-z_]+)\s*\(", src)))


def test_exports_every_declared_symbol(g):
    lib = g.load()
    names = declared_functions()
    assert len(names) >= 10
    for name in names:
        assert hasattr(lib, name), name
    assert sorted(g.EXPORTED_SYMBOLS) == names
    assert "gsofa_supernode_stitch" in names
    out = subprocess.run(["nm", "-D", "--defined-only", g.LIB_PATH], capture_output=True, text=True).stdout
    for name in names:
        assert re.search(rf"\bT {name}$", out, re.M), name


def test_struct_layout_matches_header(g):
    prog = r"""
#include <stddef.h>
#include <stdio.h>
#include "gsofa.h"
int main(void) {
  printf("%zu %zu %zu %zu\n", sizeof(gsofa_opts), sizeof(gsofa_stats), sizeof(gsofa_result),
         sizeof(gsofa_tail));
  printf("%zu %zu %zu\n", offsetof(gsofa_opts, stream), offsetof(gsofa_result, stats),
         offsetof(gsofa_result, fill_count));
  return 0;
}
"""
    with tempfile.TemporaryDirectory() as d:
        c = os.path.join(d, "t.c")
        open(c, "w").write(prog)
        exe = os.path.join(d, "t")
        subprocess.check_call(["gcc", "-std=c99", "-I", os.path.join(ROOT, "include"), c, "-o", exe])
        a, b = subprocess.check_output([exe], text=True).split("\n")[:2]
    import ctypes
    assert [int(x) for x in a.split()] == [ctypes.sizeof(g.Opts), ctypes.sizeof(g.Stats),
                                           ctypes.sizeof(g.CResult), ctypes.sizeof(g.Tail)]
    assert [int(x) for x in b.split()] == [g.Opts.stream.offset, g.CResult.stats.offset,
                                           g.CResult.fill_count.offset]


def test_version_and_strings(g):
    lib = g.load()
    assert lib.gsofa_version() == 2
    assert lib.gsofa_strerror(-2).decode() == "malformed CSR input"


def _has_gpu():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


@pytest.mark.skipif(_has_gpu(), reason="checks the no-GPU failure mode")
def test_no_gpu_fails_loudly(g):
    rp, ci = gen.paper_example()
    with pytest.raises(g.GsofaError) as e:
        g.symbolic(rp, ci)
    assert e.value.code == -5   # GSOFA_ECUDA: there is no CPU fallback


def test_partition_rows_balanced_and_aligned(g):
    rp, ci = gen.config("C5", 24)
    n = rp.size - 1
    for parts in (1, 2, 4, 8):
        b = g.partition_rows(rp, ci, parts, align=128)
        assert b[0] == 0 and b[-1] == n and np.all(np.diff(b) >= 0)
        assert np.all(b[1:-1] % 128 == 0)
    # estimated work of the 8 ranges is roughly even; the later ranges are
    # narrower because work grows with the source id
    b = g.partition_rows(rp, ci, 8, align=8)
    widths = np.diff(b)
    assert widths[0] > widths[-1]


def test_partition_rows_deterministic(g):
    rp, ci = gen.config("C4", 50)
    assert np.array_equal(g.partition_rows(rp, ci, 4), g.partition_rows(rp, ci, 4))


def test_partition_rows_rejects_bad_rowptr(g):
    """Malformed row pointers are rejected before any colidx access
    (GSOFA_EBADCSR), not read out of bounds."""
    import gen
    rp, ci = gen.random_graph(64, 0.1, seed=3)
    for bad in (lambda r: r.__setitem__(5, r[-1] + 1000),   # rowptr[i] > nnz
                lambda r: r.__setitem__(7, r[6] - 1 if r[6] > 0 else -1),  # decreasing
                lambda r: r.__setitem__(0, 1)):             # rowptr[0] != 0
        b = rp.copy()
        bad(b)
        with pytest.raises(g.GsofaError) as e:
            g.partition_rows(b, ci, 4)
        assert e.value.code == -2
