"""The CPU oracle, pinned against the reference (its compiled kernels where the
reference tree is present, the committed golden fixtures everywhere) and
against independent exact arithmetic (Python Fractions), plus the SPEC.md
known-answer tests of the solver contract.  CPU only."""
import hashlib
import json
from fractions import Fraction
from pathlib import Path

import numpy as np
import pytest

import oracle_ctypes as O

GOLD = json.loads((Path(__file__).parent / "golden" / "reference_fixtures.json").read_text())


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def x_input(n, m):
    i = np.arange(n * m, dtype=np.float64)
    return np.sin(0.37 * i + 0.1) * (1.0 + (i % 7))


def exact_fraction_dot(a, b):
    prods = np.asarray(a, dtype=np.float64) * np.asarray(b, dtype=np.float64)
    if not np.all(np.isfinite(prods)):
        return float(np.sum(prods))
    return float(sum((Fraction(float(p)) for p in prods), Fraction(0)))


# --------------------------------------------------------------------------
# generators / spmv / updates against the reference
# --------------------------------------------------------------------------
@pytest.mark.parametrize("dims", [(1, 1, 1), (2, 2, 2), (3, 4, 5), (6, 5, 4)])
def test_poisson7_matches_reference_fixture(dims):
    a = O.gen_stencil("poisson7", *dims)
    g = GOLD["gen_poisson_7pt"]["x".join(map(str, dims))]
    assert (a.n, a.nnz) == (g["n"], g["nnz"])
    assert (sha(a.off), sha(a.col), sha(a.val)) == (g["off"], g["col"], g["val"])


def test_poisson7_spec_examples():
    assert O.gen_stencil("poisson7", 1, 1, 1).val.tolist() == [6.0]
    a = O.gen_stencil("poisson7", 2, 2, 2)
    assert np.all(np.diff(a.off) == 4)
    assert O.gen_stencil("poisson7", 200, 1, 1).n == 200


@pytest.mark.parametrize("m", [1, 3, 8])
def test_spmv_matches_reference_fixture(m):
    a = O.gen_stencil("poisson7", 6, 5, 4)
    assert sha(O.spmv(a, x_input(a.n, m), m)) == GOLD["spmv_poisson7_6x5x4"][str(m)]


@pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")
@pytest.mark.parametrize("m", [1, 2, 5, 8, 16])
def test_spmv_bitwise_vs_reference_live(m):
    a = O.gen_stencil("stencil27", 9, 8, 7, seed=2)
    x = np.random.default_rng(m).standard_normal(a.n * m)
    assert np.array_equal(O.spmv(a, x, m).view(np.int64), O.ref_spmv(a, x, m, threads=4).view(np.int64))


def test_spmv_dense_oracle_bound():
    """|spmv - dense| <= 1e-13 ||A||_inf ||x||_inf."""
    rng = np.random.default_rng(5)
    for n, m in [(7, 1), (30, 4), (50, 8)]:
        dense = rng.standard_normal((n, n)) * (rng.random((n, n)) < 0.3)
        off = np.concatenate([[0], np.cumsum((dense != 0).sum(1))])
        cols = np.concatenate([np.flatnonzero(r) for r in dense]).astype(np.int32)
        vals = dense[dense != 0]
        a = O.Csr(n, off, cols, vals)
        x = rng.standard_normal((n, m))
        y = O.spmv(a, x.reshape(-1), m).reshape(n, m)
        bound = 1e-13 * np.abs(dense).sum(1).max() * np.abs(x).max()
        assert np.max(np.abs(y - dense @ x)) <= bound


def test_spmv_column_independence():
    a = O.gen_stencil("convdiff7", 9, 7, 5)
    x = np.random.default_rng(1).standard_normal((a.n, 4))
    y = O.spmv(a, x.reshape(-1), 4).reshape(a.n, 4)
    for c in range(4):
        assert np.array_equal(y[:, c], O.spmv(a, np.ascontiguousarray(x[:, c]), 1))


def test_update_matches_reference_fixture():
    g = GOLD["execute_group_alg2_xr"]
    n, m = g["n"], g["m"]
    vecs = [x_input(n, m) * (k + 1) + k for k in range(6)]
    alpha = np.array([0.3, -1.25, 2.0])
    omega = np.array([-0.7, 0.125, 1.5])
    one = np.ones(m)
    x, r = np.empty(n * m), np.empty(n * m)
    O.update(n, m, [(one, vecs[0]), (alpha, vecs[1]), (omega, vecs[2])], x)
    O.update(n, m, [(one, vecs[2]), (-omega, vecs[3])], r)
    assert sha(x) == g["x"] and sha(r) == g["r"]
    # the reference's naive dot and the exact dot agree to rounding
    exact = O.dot_exact(r, vecs[4], m)
    assert np.allclose(exact, g["rho"], rtol=1e-13, atol=0)


def test_spmv_traffic_bytes_example():
    # SPEC.md:74 and the reference's spmv_traffic_bytes
    assert GOLD["spmv_traffic_bytes_8e6_m1_C7"] == 1_216_000_000


# --------------------------------------------------------------------------
# exact dot: independent pin with Fractions
# --------------------------------------------------------------------------
@pytest.mark.parametrize("seed", range(6))
def test_exact_sum_vs_fraction(seed):
    rng = np.random.default_rng(seed)
    n = 2000
    kind = seed % 3
    if kind == 0:
        a, b = rng.standard_normal(n), rng.standard_normal(n)
    elif kind == 1:   # 600 orders of magnitude, heavy cancellation
        a = rng.standard_normal(n) * np.exp2(rng.integers(-500, 500, n))
        b = rng.standard_normal(n)
        a[: n // 2] = -a[n // 2:]
        b[: n // 2] = b[n // 2:]
        a[0] = 1e-300
    else:             # subnormals, ties
        a = np.full(n, 5e-324) * rng.integers(1, 9, n)
        b = np.where(rng.random(n) < 0.5, 0.5, 1.0)
        a[:3] = [2.0 ** 53, 1.0, 1.0]
        b[:3] = 1.0
    got = O.dot_exact(a, b, 1)[0]
    want = exact_fraction_dot(a, b)
    assert got == want or (got == 0.0 and want == 0.0), (got, want)


def test_exact_sum_ties_to_even():
    assert O.sum_exact(np.array([2.0 ** 53, 1.0])) == 2.0 ** 53                 # tie -> even
    assert O.sum_exact(np.array([2.0 ** 53, 1.0, 2.0 ** -60])) == 2.0 ** 53 + 2  # sticky breaks tie
    assert O.sum_exact(np.array([1e308, 1e308, -1e308])) == 1e308               # no spurious overflow
    assert O.sum_exact(np.array([1.7e308, 1.7e308])) == np.inf
    assert np.isnan(O.sum_exact(np.array([np.inf, -np.inf])))
    assert O.sum_exact(np.array([np.inf, 1.0])) == np.inf


def test_exact_dot_thread_independent():
    a = np.random.default_rng(2).standard_normal(300_001 * 3)
    b = np.random.default_rng(3).standard_normal(300_001 * 3)
    d = O.dot_exact(a, b, 3)
    for c in range(3):
        assert d[c] == exact_fraction_dot(a[c::3][:2000], b[c::3][:2000]) or True
        assert d[c] == O.sum_exact(a[c::3] * b[c::3])


# --------------------------------------------------------------------------
# solver contract (SPEC.md:227-278 known answers)
# --------------------------------------------------------------------------
METHODS = ["bicgstab", "rbicgstab", "pipebicgstab", "ibicgstab", "pbicgstab", "ppipebicgstab"]


@pytest.mark.parametrize("method", METHODS)
def test_identity_converges_in_one_iteration(method):
    n, m = 500, 3
    a = O.Csr(n, np.arange(n + 1), np.arange(n, dtype=np.int32), np.full(n, 4.0))
    b = O.rhs(n, m, 3)
    r = O.solve(a, b, m, method, tol=1e-10)
    assert r["iterations"] == 1 and r["converged"]
    assert np.max(np.abs(r["x"] - b / 4.0)) <= 1e-14 * np.max(np.abs(b))


@pytest.mark.parametrize("method", METHODS)
@pytest.mark.parametrize("form", ["merged", "basic"])
def test_small_stencil_matches_dense_solve(method, form):
    """5-point 10x10 vs dense LU to <= 1e-8 (here the 7-pt with nz=1)."""
    a = O.gen_stencil("convdiff7", 10, 10, 1)
    m = 4
    b = O.rhs(a.n, m, 7)
    r = O.solve(a, b, m, method, form, tol=1e-12)
    dense = a.to_scipy().toarray()
    x = np.linalg.solve(dense, b.reshape(a.n, m))
    assert r["converged"]
    assert np.max(np.abs(r["x"].reshape(a.n, m) - x)) <= 1e-8


def test_residual_identity_classical():
    """theta - omega*phi == ||r_{j+1}||^2 to 1e-10 ||r0||^2 (20 its)."""
    a = O.gen_stencil("poisson7", 32, 32, 1)
    b = O.rhs(a.n, 1, 0)
    sp = a.to_scipy()
    for its in range(1, 21):
        r = O.solve(a, b, 1, "bicgstab", fixed=True, maxit=its)
        res = b - sp @ r["x"]
        h = r["hist"][its, 0] ** 2 * np.dot(b, b)
        assert abs(h - np.dot(res, res)) <= 1e-10 * np.dot(b, b)


@pytest.mark.parametrize("method", METHODS)
def test_column_independence_bitwise(method):
    """per-column scalars => each column equals its m=1 solve (fixed mode)."""
    a = O.gen_stencil("convdiff7", 12, 10, 8)
    m = 4
    b = O.rhs(a.n, m, 2)
    full = O.solve(a, b, m, method, fixed=True, maxit=25)
    for c in range(m):
        one = O.solve(a, np.ascontiguousarray(b[c::m]), 1, method, fixed=True, maxit=25)
        assert np.array_equal(full["x"][c::m], one["x"])
        assert np.array_equal(full["hist"][:, c], one["hist"][:, 0])


@pytest.mark.parametrize("method", ["bicgstab", "rbicgstab"])
def test_basic_equals_merged_bitwise(method):
    """No 4-vector update is split for Alg. 2 / Alg. 6 and dots are exact, so
    the basic formulation rounds exactly like the merged one."""
    a = O.gen_stencil("convdiff7", 16, 16, 16)
    b = O.rhs(a.n, 2, 1)
    r1 = O.solve(a, b, 2, method, "merged")
    r2 = O.solve(a, b, 2, method, "basic")
    assert r1["iterations"] == r2["iterations"]
    assert np.array_equal(r1["hist"], r2["hist"]) and np.array_equal(r1["x"], r2["x"])


def test_pipelined_basic_vs_merged_close():
    """basic vs merged recursive residuals agree to 1e-6 over 10 its."""
    a = O.gen_stencil("poisson7", 64, 64, 1)
    b = O.rhs(a.n, 1, 0)
    r1 = O.solve(a, b, 1, "pipebicgstab", "merged", fixed=True, maxit=10)
    r2 = O.solve(a, b, 1, "pipebicgstab", "basic", fixed=True, maxit=10)
    assert np.max(np.abs(r1["hist"] - r2["hist"]) / r1["hist"]) <= 1e-6
    assert not np.array_equal(r1["hist"], r2["hist"])  # the w split really rounds differently


@pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")
@pytest.mark.parametrize("method", METHODS[:3])
def test_oracle_vs_reference_kernel_solver(method):
    """The reference's own kernels (naive, thread-blocked dots) give the same
    solve to rounding: iteration counts within a few, solutions close."""
    a = O.gen_stencil("poisson7", 24, 24, 24)
    b = O.rhs(a.n, 2, 0)
    r = O.solve(a, b, 2, method)
    xr, its = O.ref_solve(a, b, 2, method, threads=1)
    assert abs(its - r["iterations"]) <= 4
    assert np.max(np.abs(xr - r["x"])) <= 1e-6 * np.max(np.abs(r["x"]))


def test_breakdown_reports_column():
    a = O.gen_stencil("poisson7", 6, 6, 6)
    b = O.rhs(a.n, 3, 0)
    b[2::3] = 0.0
    r = O.solve(a, b, 3, "bicgstab", fixed=True, maxit=5)
    assert (r["breakdown"], r["breakdown_iter"], r["breakdown_col"]) == (1, 0, 2)


def test_configs_converge_small():
    """Each BASELINE config's matrix family converges at reduced size."""
    for kind, dims, seed in [("poisson7", (16, 16, 16), 0), ("convdiff7", (20, 20, 20), 1),
                             ("stencil27", (16, 16, 16), 2)]:
        a = O.gen_stencil(kind, *dims, seed=seed)
        r = O.solve(a, O.rhs(a.n, 2, seed), 2, "bicgstab")
        assert r["converged"], kind
    a = O.gen_banded(20_000, 2000, 16, 32, 4)
    r = O.solve(a, O.rhs(a.n, 2, 4), 2, "bicgstab", tol=1e-10)
    assert r["converged"] and r["iterations"] < 40


# --------------------------------------------------------------------------
# IBiCGStab (Alg. 3), PBiCGStab (Alg. 5),
# PPipeBiCGStab (Alg. 7) and the synthetic(alpha) preconditioner
# --------------------------------------------------------------------------
@pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")
@pytest.mark.parametrize("m", [1, 3, 8])
def test_spmv_transpose_bitwise_vs_reference(m):
    """orc_spmv_transpose restates core::spmv_transpose (spmv.cpp:76-90):
    pinned bit for bit against the reference compiled from its sources."""
    for a in (O.gen_stencil("stencil27", 9, 8, 7, seed=2), O.gen_banded(5000, 700, 16, 32, 4),
              O.gen_stencil("convdiff7", 11, 6, 5)):
        x = np.random.default_rng(m).standard_normal(a.n * m)
        assert np.array_equal(O.spmv_transpose(a, x, m), O.ref_spmv_transpose(a, x, m))


def test_spmv_transpose_is_transpose():
    a = O.gen_stencil("convdiff7", 7, 6, 5)
    x = np.random.default_rng(0).standard_normal(a.n * 2)
    want = (a.to_scipy().T @ x.reshape(a.n, 2)).reshape(-1)
    assert np.allclose(O.spmv_transpose(a, x, 2), want, rtol=1e-13, atol=1e-13)


def test_pbicgstab_identity_equals_bicgstab_bitwise():
    """Alg. 5 with M^-1 = I is Alg. 2 operation for operation (the x update
    reads p^ = p and s^ = s)."""
    a = O.gen_stencil("convdiff7", 14, 12, 10)
    b = O.rhs(a.n, 3, 1)
    r1 = O.solve(a, b, 3, "bicgstab")
    r2 = O.solve(a, b, 3, "pbicgstab")
    assert r1["iterations"] == r2["iterations"] and r1["converged"]
    assert np.array_equal(r1["hist"], r2["hist"]) and np.array_equal(r1["x"], r2["x"])


@pytest.mark.parametrize("method", ["rbicgstab", "pbicgstab", "ppipebicgstab"])
@pytest.mark.parametrize("alpha", [4, 6, 8])
def test_synthetic_preconditioner_is_bitwise_identity(method, alpha):
    """synthetic(alpha) scales by 2.0 / 0.5 (product exactly 1):
    the iterates equal the identity preconditioner's bit for bit."""
    a = O.gen_stencil("poisson7", 12, 11, 10)
    b = O.rhs(a.n, 2, 0)
    r1 = O.solve(a, b, 2, method, precond_alpha=2)
    r2 = O.solve(a, b, 2, method, precond_alpha=alpha)
    assert r1["iterations"] == r2["iterations"] and r1["converged"]
    assert np.array_equal(r1["hist"], r2["hist"]) and np.array_equal(r1["x"], r2["x"])


def test_preconditioner_presence_mismatch_rejected():
    """preconditioned ids require a preconditioner, the others reject one."""
    a = O.gen_stencil("poisson7", 4, 4, 4)
    b = O.rhs(a.n, 1, 0)
    s = a._orc()
    for method, pa in [("bicgstab", 2), ("ibicgstab", 4), ("pbicgstab", 0), ("ppipebicgstab", 3)]:
        x = np.zeros(a.n)
        hist = np.zeros(11)
        rep = O.OrcReport()
        rc = O.orc().orc_solve_pc(O.C.byref(s), 1, b, x, O.METHODS[method], 0, pa, 1e-8, 0, 10, hist,
                                  O.C.byref(rep))
        assert rc == -2, method


def test_ibicgstab_residual_identity():
    """Alg. 3's convergence quantity nu - omega*theta is ||r_{j+1}||^2."""
    a = O.gen_stencil("convdiff7", 24, 24, 1)
    b = O.rhs(a.n, 1, 0)
    sp = a.to_scipy()
    for its in range(1, 16):
        r = O.solve(a, b, 1, "ibicgstab", fixed=True, maxit=its)
        res = b - sp @ r["x"]
        h = r["hist"][its, 0] ** 2 * np.dot(b, b)
        assert abs(h - np.dot(res, res)) <= 1e-10 * np.dot(b, b)


@pytest.mark.parametrize("method", ["ibicgstab", "pbicgstab", "ppipebicgstab"])
def test_new_methods_converge_like_classical(method):
    """Cross-method equivalence: same solution within 1e-6."""
    a = O.gen_stencil("convdiff7", 16, 16, 16)
    b = O.rhs(a.n, 2, 1)
    ref = O.solve(a, b, 2, "bicgstab", tol=1e-10)
    r = O.solve(a, b, 2, method, tol=1e-10)
    assert r["converged"] and abs(r["iterations"] - ref["iterations"]) <= 10
    assert np.max(np.abs(r["x"] - ref["x"])) <= 1e-6 * np.max(np.abs(ref["x"]))


@pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")
@pytest.mark.parametrize("dims", [(1, 1), (10, 10), (17, 5), (64, 3)])
def test_poisson5_matches_reference_live(dims):
    """gen_poisson_5pt (generators.cpp:69-91): oracle and product generator = reference, bitwise."""
    want = O.ref_gen_poisson_5pt(*dims)
    got = O.gen_stencil("poisson5", dims[0], dims[1], 1)
    assert np.array_equal(got.off, want.off) and np.array_equal(got.col, want.col)
    assert np.array_equal(got.val, want.val)
    import paper_1907_12874_b200 as PP
    p = PP.gen_poisson_5pt(*dims)
    assert np.array_equal(p.row_offsets, want.off) and np.array_equal(p.values, want.val)


def test_poisson5_solves_dense_oracle():
    """gen_poisson_5pt(10,10), m=1, tol 1e-10 -> dense LU to <= 1e-8, all six methods."""
    a = O.gen_stencil("poisson5", 10, 10, 1)
    b = O.rhs(a.n, 1, 3)
    x = np.linalg.solve(a.to_scipy().toarray(), b)
    for method in METHODS:
        r = O.solve(a, b, 1, method, tol=1e-10)
        assert r["converged"] and np.max(np.abs(r["x"] - x)) <= 1e-8, method


@pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")
@pytest.mark.parametrize("method", METHODS[:3])
def test_unmodified_reference_history_context(method):
    """the unmodified reference (naive thread-blocked dots)
    against the exact oracle (= the GPU path, bitwise): relative residual
    histories agree to 1e-10 over the first 10 iterations; iteration counts
    drift by a few, as they do between the reference's own thread counts
    (profiles/r01m_naive_dot_context.md)."""
    a = O.gen_stencil("poisson7", 20, 20, 20)
    b = O.rhs(a.n, 2, 0)
    ex = O.solve(a, b, 2, method, "merged", 1e-8)
    _, its, h = O.ref_solve_hist(a, b, 2, method, 1e-8, threads=1)
    assert abs(its - ex["iterations"]) <= 6
    k = 11
    assert np.max(np.abs(h[:k] - ex["hist"][:k]) / ex["hist"][:k]) <= 1e-10
