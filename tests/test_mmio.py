"""Matrix Market ingest (host IO, no GPU): pattern CSR with the diagonal
dropped, columns ascending, symmetric storage expanded."""
import gzip

import numpy as np
import pytest

from paper_2007_00840_b200.mmio import read_matrix_market


def _write(tmp_path, text, name="a.mtx"):
    p = tmp_path / name
    if name.endswith(".gz"):
        with gzip.open(p, "wt") as f:
            f.write(text)
    else:
        p.write_text(text)
    return p


def test_general_real(tmp_path):
    p = _write(tmp_path, """%%MatrixMarket matrix coordinate real general
% a comment
4 4 6
1 1 2.0
1 3 -1
2 1 4e3
3 4 1
4 2 0.5
4 4 1
""")
    rp, ci = read_matrix_market(p)
    assert rp.tolist() == [0, 1, 2, 3, 4]
    assert ci.tolist() == [2, 0, 3, 1]           # diagonal (1,1), (4,4) dropped
    assert rp.dtype == np.int64 and ci.dtype == np.int32


def test_symmetric_pattern_expanded_and_deduplicated(tmp_path):
    p = _write(tmp_path, """%%MatrixMarket matrix coordinate pattern symmetric
3 3 4
2 1
3 1
3 2
2 1
""", "b.mtx.gz")
    rp, ci = read_matrix_market(p)
    dense = np.zeros((3, 3), int)
    for r in range(3):
        dense[r, ci[rp[r]:rp[r + 1]]] = 1
    assert (dense == np.array([[0, 1, 1], [1, 0, 1], [1, 1, 0]])).all()


def test_paper_example_round_trip(tmp_path):
    import gen
    rp0, ci0 = gen.paper_example()
    n = rp0.size - 1
    rows = np.repeat(np.arange(n), np.diff(rp0))
    body = "\n".join(f"{r + 1} {c + 1}" for r, c in zip(rows, ci0))
    p = _write(tmp_path, f"%%MatrixMarket matrix coordinate pattern general\n{n} {n} {ci0.size}\n{body}\n")
    rp, ci = read_matrix_market(p)
    assert np.array_equal(rp, rp0) and np.array_equal(ci, ci0)


@pytest.mark.parametrize("text,msg", [
    ("%%MatrixMarket matrix array real general\n2 2\n1\n2\n3\n4\n", "coordinate"),
    ("%%MatrixMarket matrix coordinate real general\n2 3 1\n1 2 1\n", "square"),
    ("%%MatrixMarket matrix coordinate real general\n2 2 2\n1 2 1\n", "expected 2"),
    ("%%MatrixMarket matrix coordinate real general\n2 2 1\n3 1 1\n", "out of range"),
])
def test_rejects_bad_files(tmp_path, text, msg):
    with pytest.raises(ValueError, match=msg):
        read_matrix_market(_write(tmp_path, text))
