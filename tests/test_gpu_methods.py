"""GPU parity for the SURVEY.md 8(f) rank-1 methods: Improved BiCGStab
(Alg. 3), preconditioned BiCGStab (Alg. 5), preconditioned Pipelined
BiCGStab (Alg. 7) and the synthetic(alpha) preconditioner,
each against the CPU oracle bit for bit (exact dots, no FMA, identical
expression trees)."""
import numpy as np
import pytest

import oracle_ctypes as O
import paper_1907_12874_b200 as P
from test_gpu_multirank_local import run_partitioned
from test_gpu_parity import assert_bitwise, assert_same_solve, to_prod

pytestmark = pytest.mark.gpu

NEW = ["ibicgstab", "pbicgstab", "ppipebicgstab"]


def run_both(ctx, a, b, m, method, form="merged", alpha=None, **kw):
    want = O.solve(a, b, m, method, form, precond_alpha=alpha, **kw)
    d = ctx.upload(to_prod(a))
    B = ctx.multivector(a.n, m, b)
    X = ctx.multivector(a.n, m)
    kw2 = dict(kw)
    if "maxit" in kw2:
        kw2["max_iters"] = kw2.pop("maxit")
    try:
        rep = P.solve(ctx, d, B, X, method, form, precond_alpha=alpha, **kw2)
    except P.BreakdownError:
        rep = None
    return want, rep, X


@pytest.mark.parametrize("form", ["merged", "basic", "fused"])
@pytest.mark.parametrize("method", NEW)
def test_new_methods_convdiff_m4(ctx, method, form):
    a = O.gen_stencil("convdiff7", 20, 18, 16)
    b = O.rhs(a.n, 4, 1)
    want, rep, X = run_both(ctx, a, b, 4, method, form)
    assert want["converged"] and want["iterations"] > 20
    assert_same_solve(want, rep, X, f"{method}/{form}")


@pytest.mark.parametrize("m", [1, 3, 8])
@pytest.mark.parametrize("method", NEW)
def test_new_methods_shapes(ctx, method, m):
    """Odd m (one column per thread) and m=1; 27-point and Poisson matrices."""
    a = O.gen_stencil("stencil27", 11, 10, 9, seed=2) if m != 1 else O.gen_stencil("poisson7", 16, 16, 16)
    b = O.rhs(a.n, m, 2)
    want, rep, X = run_both(ctx, a, b, m, method)
    assert_same_solve(want, rep, X, f"{method} m={m}")


@pytest.mark.parametrize("form", ["merged", "fused"])
@pytest.mark.parametrize("alpha", [2, 4, 6])
@pytest.mark.parametrize("method", ["rbicgstab", "pbicgstab", "ppipebicgstab"])
def test_synthetic_preconditioner(ctx, method, alpha, form):
    """identity (alpha=2) and synthetic(alpha) M^-1: same bits as the oracle,
    and the same bits as each other."""
    a = O.gen_stencil("convdiff7", 16, 14, 12)
    b = O.rhs(a.n, 2, 3)
    want, rep, X = run_both(ctx, a, b, 2, method, form, alpha=alpha)
    assert_same_solve(want, rep, X, f"{method}/{form} alpha={alpha}")
    ident = O.solve(a, b, 2, method, form, precond_alpha=2)
    assert np.array_equal(X.download(), ident["x"])


@pytest.mark.parametrize("method", NEW)
def test_new_methods_fixed_mode(ctx, method):
    a = O.gen_stencil("poisson7", 12, 12, 12)
    b = O.rhs(a.n, 2, 0)
    want, rep, X = run_both(ctx, a, b, 2, method, fixed=True, maxit=15)
    assert rep.iterations == 15
    assert_same_solve(want, rep, X, f"{method} fixed")


@pytest.mark.parametrize("method", NEW)
def test_new_methods_identity_matrix(ctx, method):
    n, m = 300, 3
    a = O.Csr(n, np.arange(n + 1), np.arange(n, dtype=np.int32), np.full(n, 4.0))
    b = O.rhs(n, m, 3)
    want, rep, X = run_both(ctx, a, b, m, method, tol=1e-10)
    assert rep.iterations == 1 and rep.converged
    assert_same_solve(want, rep, X, f"{method} identity")


def test_pbicgstab_identity_equals_bicgstab(ctx):
    a = O.gen_stencil("convdiff7", 18, 16, 14)
    b = O.rhs(a.n, 4, 1)
    d = ctx.upload(to_prod(a))
    B = ctx.multivector(a.n, 4, b)
    X1, X2 = ctx.multivector(a.n, 4), ctx.multivector(a.n, 4)
    r1 = P.solve(ctx, d, B, X1, "bicgstab")
    r2 = P.solve(ctx, d, B, X2, "pbicgstab")
    assert r1.iterations == r2.iterations
    assert_bitwise(X2.download(), X1.download(), "pbicgstab(I) vs bicgstab")


def test_traffic_counter_includes_preconditioner(ctx):
    """instrumented counts = schedule totals x iterations, plus
    the preconditioner's transfers (alpha/2 reads + alpha/2 writes each)."""
    a = O.gen_stencil("poisson7", 10, 10, 10)
    b = O.rhs(a.n, 1, 0)
    d = ctx.upload(to_prod(a))
    B = ctx.multivector(a.n, 1, b)
    for alpha in (2, 4):
        X = ctx.multivector(a.n, 1)
        rep = P.solve(ctx, d, B, X, "pbicgstab", fixed=True, max_iters=10, precond_alpha=alpha)
        s = P.method_schedule_pc("pbicgstab", "merged", alpha)
        assert rep.vector_reads == 10 * (s["reads"] + s["precond"] * alpha // 2)
        assert rep.vector_writes == 10 * (s["writes"] + s["precond"] * alpha // 2)


def test_preconditioner_presence_errors(ctx):
    a = O.gen_stencil("poisson7", 6, 6, 6)
    d = ctx.upload(to_prod(a))
    B = ctx.multivector(a.n, 1, O.rhs(a.n, 1, 0))
    X = ctx.multivector(a.n, 1)
    for method, alpha in [("bicgstab", 2), ("ibicgstab", 4), ("pbicgstab", 0), ("ppipebicgstab", 5)]:
        with pytest.raises(ValueError):
            P.solve(ctx, d, B, X, method, precond_alpha=alpha)


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("method,form", [("pbicgstab", "merged"), ("ppipebicgstab", "merged"),
                                         ("ppipebicgstab", "basic"), ("pbicgstab", "fused")])
def test_new_methods_partitioned(ctx, world, method, form):
    nx, ny, nz = 16, 14, 5 * world
    a = O.gen_stencil("convdiff7", nx, ny, nz)
    m = 4
    b = O.rhs(a.n, m, 1)
    bounds = [p * nx * ny * 5 for p in range(world + 1)]
    want = O.solve(a, b, m, method, form)
    parts = run_partitioned(a, b, m, bounds, method, form, tol=1e-8)
    for r, (rep, x) in enumerate(parts):
        assert rep.iterations == want["iterations"]
        assert np.array_equal(rep.residual_history.view(np.int64), want["hist"].view(np.int64))
        r0, r1 = bounds[r], bounds[r + 1]
        assert np.array_equal(x.view(np.int64), want["x"][r0 * m:r1 * m].view(np.int64))


def test_ibicgstab_partitioned(ctx):
    # f0 = A^T r0 across ranks (A^T halo plan built at upload), bitwise
    a = O.gen_stencil("convdiff7", 8, 8, 8)
    m = 2
    b = O.rhs(a.n, m, 1)
    want = O.solve(a, b, m, "ibicgstab", "merged", 1e-8)
    parts = run_partitioned(a, b, m, [0, 256, 512], "ibicgstab", "merged", tol=1e-8)
    for r, (rep, x) in enumerate(parts):
        assert rep.iterations == want["iterations"]
        assert np.array_equal(rep.residual_history.view(np.int64), want["hist"].view(np.int64))
        r0, r1 = [0, 256, 512][r], [0, 256, 512][r + 1]
        assert np.array_equal(x.view(np.int64), want["x"][r0 * m:r1 * m].view(np.int64))


def test_matrix_market_ingest_partitioned(ctx, tmp_path):
    """a MatrixMarket file (arbitrary sparsity) ->
    device CSR with the general halo plan over uneven row blocks -> the same
    bits as the single-GPU / oracle solve."""
    a = O.gen_banded(30_000, 9_000, 8, 20, 4)
    path = tmp_path / "band.mtx"
    P.write_matrix_market(P.CsrMatrix(a.n, a.off, a.col, a.val), path)
    m_ = P.read_matrix_market(path)
    assert np.array_equal(m_.values.view(np.int64), a.val.view(np.int64))
    a2 = O.Csr(m_.n_rows, m_.row_offsets, m_.col_indices, m_.values)
    m = 4
    b = O.rhs(a2.n, m, 4)
    bounds = [0, 7_001, 19_500, 30_000]
    want = O.solve(a2, b, m, "pipebicgstab", fixed=True, maxit=20)
    parts = run_partitioned(a2, b, m, bounds, "pipebicgstab", "merged", fixed=True, max_iters=20)
    for r, (rep, x) in enumerate(parts):
        assert rep.iterations == 20
        assert np.array_equal(rep.residual_history.view(np.int64), want["hist"].view(np.int64))
        assert np.array_equal(x.view(np.int64), want["x"][bounds[r] * m:bounds[r + 1] * m].view(np.int64))


def test_fusion_bench_runs_agree(ctx):
    """Fig. 2: run #3 (three updates in one pass) computes exactly what run #1
    (three passes) computes; the merged runs move 5N instead of 9N elements."""
    r = P.fusion_bench(ctx, n=1 << 22, reps=3)
    assert r["run3_equals_run1"]
    assert all(t > 0 for t in r["ms"])


@pytest.mark.parametrize("form", ["merged", "fused"])
@pytest.mark.parametrize("method", ["bicgstab", "rbicgstab", "pipebicgstab", "ibicgstab", "pbicgstab",
                                    "ppipebicgstab"])
def test_grid_reordered_operator_bitwise(ctx, method, form):
    """mbg_csr_set_grid: the solver works on a brick-reordered P A P^T (each
    row summed in its original order; A^T for IBiCGStab built in the original
    order) -- iterates, history and x must equal the oracle bit for bit."""
    nx, ny, nz = 13, 11, 10
    a = O.gen_stencil("stencil27", nx, ny, nz, seed=2)
    m = 4
    b = O.rhs(a.n, m, 2)
    want = O.solve(a, b, m, method, form)
    d = ctx.upload(to_prod(a))
    assert d.set_grid(nx, ny, nz)
    B = ctx.multivector(a.n, m, b)
    X = ctx.multivector(a.n, m)
    rep = P.solve(ctx, d, B, X, method, form)
    assert_same_solve(want, rep, X, f"reordered {method}/{form}")
    # the SpMV entry point still applies the caller's operator
    Y = ctx.multivector(a.n, m)
    P.spmv(ctx, d, B, Y)
    assert_bitwise(Y.download(), O.spmv(a, b, m), "spmv after set_grid")


def test_grid_hint_ignored_for_short_rows(ctx):
    a = O.gen_stencil("convdiff7", 12, 10, 8)
    d = ctx.upload(to_prod(a))
    assert not d.set_grid(12, 10, 8)
    with pytest.raises(ValueError):
        d.set_grid(12, 10, 9)


@pytest.mark.parametrize("method", ["bicgstab", "ibicgstab", "ppipebicgstab"])
def test_true_residual_after_solve(ctx, method):
    """The recomputed ||b - Ax|| / ||b|| of a converged solve is small and
    agrees with a host double-precision evaluation."""
    a = O.gen_stencil("convdiff7", 16, 14, 12)
    m = 3
    b = O.rhs(a.n, m, 1)
    d = ctx.upload(to_prod(a))
    B = ctx.multivector(a.n, m, b)
    X = ctx.multivector(a.n, m)
    rep = P.solve(ctx, d, B, X, method, tol=1e-10)
    tr = P.true_residual(ctx, d, B, X)
    x = X.download().reshape(a.n, m)
    r = b.reshape(a.n, m) - a.to_scipy() @ x
    host = np.linalg.norm(r, axis=0) / np.linalg.norm(b.reshape(a.n, m), axis=0)
    assert rep.converged and np.all(tr < 1e-8)
    assert np.allclose(tr, host, rtol=1e-6, atol=1e-14)


@pytest.mark.parametrize("m", [3, 5])
@pytest.mark.parametrize("form", ["basic", "merged", "fused"])
@pytest.mark.parametrize("method", ["bicgstab", "pbicgstab"])
def test_multi_trip_tails(ctx, method, form, m):
    """Odd m at ~150k rows: the one-column-per-thread passes run several grid-stride trips of
    4 packets with a partial last trip (dot1 / dot2 / upd2_sq / pbcg_r) -- same bits."""
    a = O.gen_stencil("poisson7", 53, 53, 53)
    b = O.rhs(a.n, m, 4)
    want, rep, X = run_both(ctx, a, b, m, method, form, fixed=True, maxit=12)
    assert rep.iterations == 12
    assert_same_solve(want, rep, X, f"{method}/{form} m={m}")
