"""MatrixMarket ingest against the reference's own
reader (proj/src/core/matrix_market.cpp, compiled into oracle/_ref): same
arrays bit for bit, same "<name>:<line>: message" errors, SPEC.md:83-91
examples; the write side round-trips exactly (%.17g)."""
import numpy as np
import pytest

import oracle_ctypes as O
import paper_1907_12874_b200 as P

needs_ref = pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")


def same(a: P.CsrMatrix, b: O.Csr):
    assert a.n_rows == b.n
    assert np.array_equal(a.row_offsets, b.off)
    assert np.array_equal(a.col_indices, b.col)
    assert np.array_equal(a.values.view(np.int64), b.val.view(np.int64))


def write(tmp_path, name, text):
    p = tmp_path / name
    p.write_text(text)
    return p


def test_identity_2x2(tmp_path):
    p = write(tmp_path, "i.mtx", "%%MatrixMarket matrix coordinate real general\n2 2 2\n1 1 1.0\n2 2 1.0\n")
    a = P.read_matrix_market(p)
    assert list(a.row_offsets) == [0, 1, 2] and list(a.col_indices) == [0, 1]


def test_symmetric_expansion_and_duplicates(tmp_path):
    # lower triangle of a 4x4 symmetric matrix, one duplicated (2,1) entry
    p = write(tmp_path, "s.mtx", "%%MatrixMarket matrix coordinate real symmetric\n% comment\n\n4 4 6\n"
                                 "1 1 4\n2 1 -1.5\n2 1 0.25\n3 2 -1\n4 4 2\n4 1 0.5\n")
    a = P.read_matrix_market(p)
    dense = np.zeros((4, 4))
    for i in range(4):
        for k in range(a.row_offsets[i], a.row_offsets[i + 1]):
            dense[i, a.col_indices[k]] = a.values[k]
    assert np.array_equal(dense, dense.T) and dense[1, 0] == -1.25 and dense[3, 0] == 0.5
    assert a.nnz() == 2 * 6 - 2 - 1 - 1   # expansion doubles off-diagonals; duplicate merged


@needs_ref
@pytest.mark.parametrize("sym", ["general", "symmetric"])
@pytest.mark.parametrize("field", ["real", "integer"])
def test_bitwise_vs_reference_reader(tmp_path, sym, field):
    rng = np.random.default_rng(5)
    n = 300
    lines = []
    for _ in range(2500):
        i, j = rng.integers(1, n + 1, 2)
        if sym == "symmetric" and j > i:
            i, j = j, i
        v = int(rng.integers(-9, 10)) if field == "integer" else float(rng.standard_normal() * 10.0 ** int(rng.integers(-5, 5)))
        lines.append(f"{i} {j} {v!r}" if field == "real" else f"{i} {j} {v}")
    # distinct (row, col) pairs only: the reference's duplicate order is unspecified
    seen, uniq = set(), []
    for ln in lines:
        i, j, _ = ln.split()
        if (i, j) not in seen:
            seen.add((i, j))
            uniq.append(ln)
    text = f"%%MatrixMarket matrix coordinate {field} {sym}\n%c\n{n} {n} {len(uniq)}\n" + "\n".join(uniq) + "\n"
    p = write(tmp_path, "r.mtx", text)
    same(P.read_matrix_market(p), O.ref_read_matrix_market(p))


@needs_ref
def test_duplicates_summed_like_reference(tmp_path):
    # dyadic values: the sum is exact in any order, so the readers must agree
    p = write(tmp_path, "d.mtx", "%%MatrixMarket matrix coordinate real general\n3 3 7\n"
                                 "1 1 0.5\n3 2 1.25\n1 1 0.25\n2 3 -2\n3 2 -0.125\n1 1 4\n2 2 1\n")
    same(P.read_matrix_market(p), O.ref_read_matrix_market(p))


@needs_ref
def test_generated_matrix_roundtrip(tmp_path):
    a = O.gen_stencil("stencil27", 9, 8, 7, seed=2)
    p = tmp_path / "g.mtx"
    O.ref_write_matrix_market(a, p)
    same(P.read_matrix_market(p), a)
    q = tmp_path / "h.mtx"
    P.write_matrix_market(P.read_matrix_market(p), q)
    assert q.read_text() == p.read_text()


BAD = [
    ("", None),
    ("%%MatrixMarket matrix array real general\n2 2\n", None),
    ("%MatrixMarket matrix coordinate real general\n", None),
    ("%%MatrixMarket vector coordinate real general\n", None),
    ("%%MatrixMarket matrix coordinate complex general\n", None),
    ("%%MatrixMarket matrix coordinate real hermitian\n", None),
    ("%%MatrixMarket matrix coordinate real general\n%only comments\n", None),
    ("%%MatrixMarket matrix coordinate real general\n2 x 2\n", None),
    ("%%MatrixMarket matrix coordinate real general\n2 3 1\n1 1 1\n", None),
    ("%%MatrixMarket matrix coordinate real general\n0 0 0\n", None),
    ("%%MatrixMarket matrix coordinate real general\n2 2 2\n1 1 1\n", None),
    ("%%MatrixMarket matrix coordinate real general\n2 2 2\n1 1 1\n\n% c\n2 two 1\n", None),
    ("%%MatrixMarket matrix coordinate real general\n2 2 2\n1 1 1\n3 1 1\n", None),
    ("%%MatrixMarket matrix coordinate real general\n2 2 1\n1 1 1\n3 1 oops\n", "ok"),  # past ne: ignored
]


@needs_ref
@pytest.mark.parametrize("k", range(len(BAD)))
def test_errors_match_reference(tmp_path, k):
    text, ok = BAD[k]
    p = write(tmp_path, f"bad{k}.mtx", text)
    if ok:
        same(P.read_matrix_market(p), O.ref_read_matrix_market(p))
        return
    with pytest.raises(RuntimeError) as ref_err:
        O.ref_read_matrix_market(p)
    with pytest.raises(RuntimeError) as our_err:
        P.read_matrix_market(p)
    assert str(our_err.value) == str(ref_err.value)


def test_missing_file():
    with pytest.raises(RuntimeError, match="cannot open file"):
        P.read_matrix_market("/nonexistent/x.mtx")
