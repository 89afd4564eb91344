"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle.

Bar: bit-exact.  SpMV and updates round every multiply
and add exactly like the reference kernels; dots are exact on both sides; so
solution vectors, residual histories and iteration counts must be identical.
"""
import numpy as np
import pytest

import oracle_ctypes as O
import paper_1907_12874_b200 as P

pytestmark = pytest.mark.gpu


def to_prod(a: O.Csr) -> P.CsrMatrix:
    return P.CsrMatrix(a.n, a.off, a.col, a.val)


def bits(x):
    return np.ascontiguousarray(x, dtype=np.float64).view(np.int64)


def assert_bitwise(got, want, what=""):
    g, w = bits(got), bits(want)
    if not np.array_equal(g, w):
        bad = np.flatnonzero(g != w)
        raise AssertionError(f"{what}: {bad.size} of {g.size} differ; first {bad[:5]}: "
                             f"{np.asarray(got).reshape(-1)[bad[:5]]} vs {np.asarray(want).reshape(-1)[bad[:5]]}")


MATRICES = {
    "poisson7_16": lambda: O.gen_stencil("poisson7", 16, 16, 16),
    "convdiff_24x20x9": lambda: O.gen_stencil("convdiff7", 24, 20, 9),
    "stencil27_13": lambda: O.gen_stencil("stencil27", 13, 11, 10, seed=2),
    "banded_50k": lambda: O.gen_banded(50_000, 4096, 16, 32, 4),
}


@pytest.mark.parametrize("mname", list(MATRICES))
@pytest.mark.parametrize("m", [1, 2, 3, 4, 8, 16, 32])
def test_spmv_bitwise(ctx, mname, m):
    a = MATRICES[mname]()
    x = np.random.default_rng(m).standard_normal(a.n * m)
    want = O.spmv(a, x, m)
    d = ctx.upload(to_prod(a))
    X = ctx.multivector(a.n, m, x)
    Y = ctx.multivector(a.n, m)
    P.spmv(ctx, d, X, Y)
    assert_bitwise(Y.download(), want, f"spmv {mname} m={m}")


def test_spmv_empty_and_ragged_rows(ctx):
    # rows with 0, 1 and 40 nonzeros, one empty row at the end
    n = 300
    rng = np.random.default_rng(7)
    off, cols, vals = [0], [], []
    for i in range(n):
        k = [0, 1, 40, 3][i % 4] if i < n - 1 else 0
        c = np.sort(rng.choice(n, size=k, replace=False)).astype(np.int32)
        cols.extend(c)
        vals.extend(rng.standard_normal(k))
        off.append(len(cols))
    a = O.Csr(n, np.array(off), np.array(cols, np.int32), np.array(vals))
    for m in (1, 8, 5):
        x = rng.standard_normal(n * m)
        d = ctx.upload(to_prod(a))
        X, Y = ctx.multivector(n, m, x), ctx.multivector(n, m)
        P.spmv(ctx, d, X, Y)
        assert_bitwise(Y.download(), O.spmv(a, x, m), f"ragged m={m}")


def test_spmv_errors(ctx):
    a = O.gen_stencil("poisson7", 4, 4, 4)
    d = ctx.upload(to_prod(a))
    X = ctx.multivector(a.n, 2)
    with pytest.raises(ValueError, match="distinct storage"):
        P.spmv(ctx, d, X, X)
    with pytest.raises(ValueError, match="dimension mismatch"):
        P.spmv(ctx, d, X, ctx.multivector(a.n, 3))


@pytest.mark.parametrize("m", [1, 4, 8, 6, 32])
def test_execute_group_fused(ctx, m):
    """Alg. 2 line 15 group: x = x + a p + w s; r = s - w t; rho = (r, r0) -- bitwise."""
    n = 20_011
    rng = np.random.default_rng(m)
    vecs = [rng.standard_normal(n * m) for _ in range(6)]  # x p s t r0 r
    alpha, omega = rng.standard_normal(m), rng.standard_normal(m)
    one = np.ones(m)
    grp = [P.UpdateStatement(0, [(one, 0), (alpha, 1), (omega, 2)]),
           P.UpdateStatement(5, [(one, 2), (-omega, 3)]),
           P.DotStatement(5, 4, 0), P.DotStatement(3, 3, 1)]
    dev = [ctx.multivector(n, m, v) for v in vecs]
    dots = P.execute_group(ctx, grp, dev)
    x = np.empty_like(vecs[0]); r = np.empty_like(vecs[0])
    O.update(n, m, [(one, vecs[0]), (alpha, vecs[1]), (omega, vecs[2])], x)
    O.update(n, m, [(one, vecs[2]), (-omega, vecs[3])], r)
    assert_bitwise(dev[0].download(), x, "x")
    assert_bitwise(dev[5].download(), r, "r")
    assert_bitwise(dots[0], O.dot_exact(r, vecs[4], m), "rho")
    assert_bitwise(dots[1], O.dot_exact(vecs[3], vecs[3], m), "(t,t)")


def test_execute_group_exact_dot_adversarial(ctx):
    """Cancellation across 600 orders of magnitude, subnormals and ties."""
    m = 2
    n = 4096
    rng = np.random.default_rng(3)
    a = rng.standard_normal(n * m) * np.exp2(rng.integers(-600, 600, n * m))
    b = rng.standard_normal(n * m)
    a[:10] = 1e300; b[:10] = 1.0
    a[10:20] = -1e300; b[10:20] = 1.0
    a[20:30] = 5e-324; b[20:30] = 0.75
    dev = [ctx.multivector(n, m, a), ctx.multivector(n, m, b)]
    dots = P.execute_group(ctx, [P.DotStatement(0, 1, 0)], dev)
    assert_bitwise(dots[0], O.dot_exact(a, b, m), "adversarial")


def test_execute_group_nonfinite(ctx):
    m, n = 3, 1000
    a = np.ones(n * m); b = np.ones(n * m)
    a[0] = np.inf          # column 0: +inf
    a[1] = np.inf; a[4] = -np.inf   # column 1: inf - inf -> nan
    a[5] = np.nan          # column 2: nan
    dev = [ctx.multivector(n, m, a), ctx.multivector(n, m, b)]
    d = P.execute_group(ctx, [P.DotStatement(0, 1, 0)], dev)[0]
    assert d[0] == np.inf and np.isnan(d[1]) and np.isnan(d[2])


def test_execute_group_errors(ctx):
    n, m = 10, 2
    v = [ctx.multivector(n, m), ctx.multivector(n, 3)]
    with pytest.raises(ValueError, match="unbound vector id"):
        P.execute_group(ctx, [P.DotStatement(0, 5, 0)], v)
    with pytest.raises(ValueError, match="shape mismatch"):
        P.execute_group(ctx, [P.DotStatement(0, 1, 0)], v)
    assert P.execute_group(ctx, [], v, nslots=0).size == 0


# ---------------------------------------------------------------------------
# whole solves
# ---------------------------------------------------------------------------
def run_both(ctx, a, b, m, method, formulation="merged", tol=1e-8, fixed=False, maxit=1000, graph=True):
    want = O.solve(a, b, m, method, formulation, tol, fixed, maxit)
    d = ctx.upload(to_prod(a))
    B = ctx.multivector(a.n, m, b)
    X = ctx.multivector(a.n, m)
    try:
        rep = P.solve(ctx, d, B, X, method, formulation, tol, fixed, maxit)
    except P.BreakdownError:
        rep = None
    return want, rep, X


def assert_same_solve(want, rep, X, what):
    assert rep is not None, f"{what}: GPU reported breakdown, oracle {want['breakdown']}"
    assert rep.iterations == want["iterations"], f"{what}: iterations {rep.iterations} vs {want['iterations']}"
    assert rep.converged == want["converged"], what
    assert_bitwise(rep.residual_history, want["hist"], f"{what} history")
    assert_bitwise(X.download(), want["x"], f"{what} x")


METHODS = [(m, f) for m in ("bicgstab", "rbicgstab", "pipebicgstab") for f in ("merged", "basic", "fused")]


@pytest.mark.parametrize("method,form", METHODS)
def test_solve_config1_poisson32(ctx, method, form):
    """BASELINE config 1: Poisson 32^3, m=1, seed 0, tol 1e-8, max 1000."""
    a = O.gen_stencil("poisson7", 32, 32, 32)
    b = O.rhs(a.n, 1, 0)
    want, rep, X = run_both(ctx, a, b, 1, method, form)
    assert want["converged"] and want["iterations"] > 50
    assert_same_solve(want, rep, X, f"C1 {method}/{form}")


@pytest.mark.parametrize("method,form", METHODS)
def test_solve_convdiff_m8(ctx, method, form):
    """Config-2 shape at 40^3 (conv-diff, m=8, seed 1)."""
    a = O.gen_stencil("convdiff7", 40, 40, 40)
    b = O.rhs(a.n, 8, 1)
    want, rep, X = run_both(ctx, a, b, 8, method, form)
    assert want["converged"]
    assert_same_solve(want, rep, X, f"convdiff {method}/{form}")


@pytest.mark.parametrize("form", ["merged", "fused"])
@pytest.mark.parametrize("method", ["bicgstab", "rbicgstab", "pipebicgstab"])
def test_solve_stencil27_m16(ctx, method, form):
    """Config-3 shape at 24^3 (27-pt perturbed, m=16, seed 2)."""
    a = O.gen_stencil("stencil27", 24, 24, 24, seed=2)
    b = O.rhs(a.n, 16, 2)
    want, rep, X = run_both(ctx, a, b, 16, method, form)
    assert_same_solve(want, rep, X, f"27pt {method}/{form}")


@pytest.mark.parametrize("form", ["merged", "fused"])
@pytest.mark.parametrize("method", ["bicgstab", "rbicgstab", "pipebicgstab"])
def test_solve_fixed_m32(ctx, method, form):
    """Config-4 shape at 32^3: conv-diff, m=32, fixed 40 iterations."""
    a = O.gen_stencil("convdiff7", 32, 32, 32)
    b = O.rhs(a.n, 32, 3)
    want, rep, X = run_both(ctx, a, b, 32, method, form, fixed=True, maxit=40)
    assert want["iterations"] == 40
    assert_same_solve(want, rep, X, f"fixed m32 {method}/{form}")


@pytest.mark.parametrize("form", ["merged", "fused"])
@pytest.mark.parametrize("m", [1, 2, 3, 8])
@pytest.mark.parametrize("method", ["bicgstab", "rbicgstab", "pipebicgstab"])
def test_solve_banded(ctx, method, m, form):
    """Config-5 shape at n=100k (random banded, seed 4), fixed 30 iterations."""
    if form == "fused" and m == 3:
        pytest.skip("fused SpMM epilogue needs m in {1,2,4,8,16,32}")
    a = O.gen_banded(100_000, 65536, 16, 32, 4)
    b = O.rhs(a.n, m, 4)
    want, rep, X = run_both(ctx, a, b, m, method, form, fixed=True, maxit=30)
    assert_same_solve(want, rep, X, f"banded {method}/{form} m={m}")


def test_spmv_long_rows(ctx):
    """Rows longer than a SpMM tile's shared-memory capacity (read from global)."""
    n = 3000
    rng = np.random.default_rng(5)
    lens = np.where(np.arange(n) % 500 == 7, 2000, 5)
    off = np.concatenate([[0], np.cumsum(lens)])
    cols = np.concatenate([np.sort(rng.choice(n, size=k, replace=False)) for k in lens]).astype(np.int32)
    a = O.Csr(n, off, cols, rng.standard_normal(off[-1]))
    for m in (1, 2, 8, 32):
        x = rng.standard_normal(n * m)
        d = ctx.upload(to_prod(a))
        X, Y = ctx.multivector(n, m, x), ctx.multivector(n, m)
        P.spmv(ctx, d, X, Y)
        assert_bitwise(Y.download(), O.spmv(a, x, m), f"long rows m={m}")


def test_solve_breakdown_zero_rhs_column(ctx):
    a = O.gen_stencil("poisson7", 8, 8, 8)
    b = O.rhs(a.n, 2, 0)
    b[1::2] = 0.0   # column 1 is zero -> delta = 0 at iteration 0
    want = O.solve(a, b, 2, "bicgstab", fixed=True, maxit=10)
    assert want["breakdown"] == 1 and want["breakdown_col"] == 1 and want["breakdown_iter"] == 0
    d = ctx.upload(to_prod(a))
    B, X = ctx.multivector(a.n, 2, b), ctx.multivector(a.n, 2)
    with pytest.raises(P.BreakdownError, match="iteration 0, column 1"):
        P.solve(ctx, d, B, X, "bicgstab", fixed=True, max_iters=10)


def test_solve_identity_one_iteration(ctx):
    """A = diagonal => converges within one iteration."""
    n, m = 1000, 3
    a = O.Csr(n, np.arange(n + 1), np.arange(n, dtype=np.int32), np.full(n, 4.0))
    b = O.rhs(n, m, 9)
    for method in ("bicgstab", "rbicgstab", "pipebicgstab"):
        want, rep, X = run_both(ctx, a, b, m, method, tol=1e-10)
        assert want["iterations"] == 1
        assert_same_solve(want, rep, X, f"identity {method}")
        assert np.max(np.abs(X.download() - b / 4.0)) <= 1e-14


def test_solve_zero_iterations(ctx):
    a = O.gen_stencil("poisson7", 6, 6, 6)
    b = O.rhs(a.n, 2, 1)
    want, rep, X = run_both(ctx, a, b, 2, "bicgstab", fixed=True, maxit=0)
    assert rep.iterations == 0 == want["iterations"]
    assert_bitwise(rep.residual_history, want["hist"], "h0")


def test_solve_host_matches_device(ctx):
    a = O.gen_stencil("convdiff7", 20, 20, 20)
    m = 4
    b = O.rhs(a.n, m, 1)
    d = ctx.upload(to_prod(a))
    x = np.zeros(a.n * m)
    rep = P.solve_host(ctx, d, b, x, m, "pipebicgstab")
    want = O.solve(a, b, m, "pipebicgstab")
    assert rep.iterations == want["iterations"]
    assert_bitwise(x, want["x"], "host x")
    assert_bitwise(rep.residual_history, want["hist"], "host hist")


def test_graph_replay_overshoot_is_noop(ctx):
    """Iterations after convergence (graph chunk overshoot) must not touch x."""
    a = O.gen_stencil("poisson7", 10, 10, 10)
    b = O.rhs(a.n, 1, 0)
    want, rep, X = run_both(ctx, a, b, 1, "bicgstab", maxit=1000)
    assert rep.iterations < 64 and rep.gpu_launches > 0
    assert_same_solve(want, rep, X, "overshoot")


def test_solve_host_pinned_buffers(ctx):
    """Page-locked host buffers take the direct-DMA path of mbg_solve_host."""
    a = O.gen_stencil("convdiff7", 20, 18, 16)
    m = 4
    b = O.rhs(a.n, m, 1)
    want = O.solve(a, b, m, "bicgstab")
    d = ctx.upload(to_prod(a))
    bp = P.pinned_empty(a.n * m)
    bp[:] = b
    xp = P.pinned_empty(a.n * m)
    xp[:] = 0.0
    rep = P.solve_host(ctx, d, bp, xp, m, "bicgstab")
    assert rep.iterations == want["iterations"]
    assert_bitwise(xp, want["x"], "pinned solve_host x")


@pytest.mark.parametrize("method,form", [("bicgstab", "fused"), ("bicgstab", "merged"), ("pipebicgstab", "fused"),
                                         ("rbicgstab", "merged"), ("ibicgstab", "merged")])
def test_solve_overflowing_dots_match_oracle(ctx, method, form):
    """Products overflowing to inf (column 0 scaled by 1e200) take the
    streaming kernels' careful recomputation path; NaN in another column
    poisons only that column's dots.  The GPU must follow the oracle exactly."""
    a = O.gen_stencil("poisson7", 10, 9, 8)
    m = 3
    b = O.rhs(a.n, m, 0)
    b[0::m] *= 1e200
    b[5 * m + 2] = np.nan
    want, rep, X = run_both(ctx, a, b, m, method, form, fixed=True, maxit=6)
    if rep is None:
        assert want["breakdown"] != 0
        return
    assert rep.iterations == want["iterations"]
    assert_bitwise(rep.residual_history, want["hist"], f"{method}/{form} overflow history")
    assert_bitwise(X.download(), want["x"], f"{method}/{form} overflow x")


@pytest.mark.parametrize("mname", list(MATRICES))
@pytest.mark.parametrize("m", [1, 3, 8])
def test_spmv_transpose_bitwise(ctx, mname, m):
    """core::spmv_transpose: the oracle (pinned to the compiled reference) bit for bit."""
    a = MATRICES[mname]()
    x = np.random.default_rng(50 + m).standard_normal(a.n * m)
    d = ctx.upload(to_prod(a))
    X = ctx.multivector(a.n, m, x)
    Y = ctx.multivector(a.n, m)
    P.spmv_transpose(ctx, d, X, Y)
    assert_bitwise(Y.download(), O.spmv_transpose(a, x, m), f"spmv_transpose {mname} m={m}")


def test_too_many_columns_rejected(ctx):
    a = O.gen_stencil("poisson7", 4, 4, 4)
    d = ctx.upload(to_prod(a))
    m = 300
    B = ctx.multivector(a.n, m, np.ones(a.n * m))
    X = ctx.multivector(a.n, m)
    with pytest.raises(ValueError, match="256"):
        P.solve(ctx, d, B, X, "bicgstab")
    # the SpMM itself takes any m (generic kernel)
    Y = ctx.multivector(a.n, m)
    P.spmv(ctx, d, B, Y)
    assert_bitwise(Y.download(), O.spmv(a, np.ones(a.n * m), m), "spmv m=300")


def test_empty_inputs(ctx):
    """0 rows and 0 nonzeros: spmv writes zeros, dots over no element are +0 (the
    reference's loops simply do not run: spmv.cpp:54-74, execute.cpp:123-172)."""
    m = 4
    # n > 0, no nonzero at all
    n = 37
    a = O.Csr(n, np.zeros(n + 1, np.int64), np.zeros(0, np.int32), np.zeros(0))
    d = ctx.upload(to_prod(a))
    X = ctx.multivector(n, m, np.random.default_rng(0).standard_normal(n * m))
    Y = ctx.multivector(n, m, np.full(n * m, 7.0))
    P.spmv(ctx, d, X, Y)
    assert_bitwise(Y.download(), O.spmv(a, X.download(), m), "nnz = 0")
    # 0 rows
    a0 = O.Csr(0, np.zeros(1, np.int64), np.zeros(0, np.int32), np.zeros(0))
    d0 = ctx.upload(to_prod(a0))
    X0, Y0 = ctx.multivector(0, m), ctx.multivector(0, m)
    # two empty std::vectors share data() == nullptr, so the reference's storage check
    # (spmv.cpp:20-25) rejects a 0-row spmv; so does the device path
    with pytest.raises(ValueError, match="distinct storage"):
        P.spmv(ctx, d0, X0, Y0)
    dev = [ctx.multivector(0, m), ctx.multivector(0, m)]
    one = np.ones(m)
    dots = P.execute_group(ctx, [P.UpdateStatement(1, [(one, 0)]), P.DotStatement(0, 1, 0)], dev)
    assert np.array_equal(np.asarray(dots[0]), np.zeros(m))
    assert not np.signbit(np.asarray(dots[0])).any()


@pytest.mark.parametrize("m", [1, 3, 8])
def test_execute_group_write_through(ctx, m):
    """Statements see the outputs of earlier statements of the same group, including an
    input overwritten in place (execute.cpp:97-119): u = a + c b ; a = a - d u ;
    dots (a, u), (u, u), (b, a) into slots 2, 0, 1."""
    n = 5_003
    rng = np.random.default_rng(11 + m)
    a, b = rng.standard_normal(n * m), rng.standard_normal(n * m)
    c, dd = rng.standard_normal(m), rng.standard_normal(m)
    one = np.ones(m)
    dev = [ctx.multivector(n, m, a), ctx.multivector(n, m, b), ctx.multivector(n, m)]
    grp = [P.UpdateStatement(2, [(one, 0), (c, 1)]),
           P.UpdateStatement(0, [(one, 0), (-dd, 2)]),
           P.DotStatement(0, 2, 2), P.DotStatement(2, 2, 0), P.DotStatement(1, 0, 1)]
    dots = P.execute_group(ctx, grp, dev, nslots=3)
    u = np.empty_like(a)
    O.update(n, m, [(one, a), (c, b)], u)
    a2 = np.empty_like(a)
    O.update(n, m, [(one, a), (-dd, u)], a2)
    assert_bitwise(dev[2].download(), u, "u")
    assert_bitwise(dev[0].download(), a2, "a in place")
    assert_bitwise(dots[2], O.dot_exact(a2, u, m), "(a, u)")
    assert_bitwise(dots[0], O.dot_exact(u, u, m), "(u, u)")
    assert_bitwise(dots[1], O.dot_exact(b, a2, m), "(b, a)")


@pytest.mark.gpu
@pytest.mark.parametrize("reserve", [4, 37])
def test_reserved_sms_bitwise(reserve):
    # persistent grids sized for fewer SMs (what a multi-rank NCCL context does
    # to leave room for side-stream collectives) give the same bits
    a = O.gen_stencil("stencil27", 40, 24, 20, seed=2)
    m = 16
    b = O.rhs(a.n, m, 2)
    want = O.solve(a, b, m, "rbicgstab", "merged", 1e-8, fixed=True, maxit=12)
    c = P.Context(0)
    c.reserve_sms(reserve)
    for grid in (False, True):
        d = c.upload(to_prod(a))
        if grid:
            d.set_grid(40, 24, 20)
        B, X = c.multivector(a.n, m, b), c.multivector(a.n, m)
        rep = P.solve(c, d, B, X, "rbicgstab", "fused", 1e-8, fixed=True, max_iters=12)
        assert_bitwise(rep.residual_history, want["hist"], f"reserve {reserve} history")
        assert_bitwise(X.download(), want["x"], f"reserve {reserve} x")
    c.close()
