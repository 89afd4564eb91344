"""The one-launch classical loop for small systems (small.cu) against the
oracle and against the multi-kernel path: bitwise, converge and fixed modes,
merged and fused formulations, several m, breakdown reporting."""
import numpy as np
import pytest

import oracle_ctypes as O
import paper_1907_12874_b200 as P
from test_gpu_parity import assert_bitwise, to_prod

pytestmark = pytest.mark.gpu


def run(ctx, a, b, m, form, small, **kw):
    ctx.set_small_path(small)
    try:
        d = ctx.upload(to_prod(a))
        B, X = ctx.multivector(a.n, m, b), ctx.multivector(a.n, m)
        l0 = ctx.launches()
        rep = P.solve(ctx, d, B, X, "bicgstab", form, **kw)
        return rep, X.download(), ctx.launches() - l0
    finally:
        ctx.set_small_path(True)


@pytest.mark.parametrize("form", ["merged", "fused"])
@pytest.mark.parametrize("m", [1, 2, 8, 32])
def test_small_loop_bitwise(ctx, form, m):
    a = O.gen_stencil("poisson7", 16, 12, 10)
    b = O.rhs(a.n, m, 0)
    want = O.solve(a, b, m, "bicgstab", form, 1e-8)
    rep, x, launches = run(ctx, a, b, m, form, True, tol=1e-8)
    assert rep.iterations == want["iterations"] and rep.converged == want["converged"]
    assert_bitwise(rep.residual_history, want["hist"], "small history")
    assert_bitwise(x, want["x"], "small x")
    rep2, x2, launches2 = run(ctx, a, b, m, form, False, tol=1e-8)
    assert_bitwise(rep2.residual_history, rep.residual_history, "multi-kernel vs small")
    assert_bitwise(x2, x, "multi-kernel vs small x")
    assert launches < launches2   # the loop is one launch


def test_small_loop_fixed_and_convdiff(ctx):
    a = O.gen_stencil("convdiff7", 20, 20, 20, seed=1)
    m = 4
    b = O.rhs(a.n, m, 1)
    want = O.solve(a, b, m, "bicgstab", "merged", fixed=True, maxit=37)
    rep, x, _ = run(ctx, a, b, m, "merged", True, fixed=True, max_iters=37)
    assert rep.iterations == 37
    assert_bitwise(rep.residual_history, want["hist"], "fixed history")
    assert_bitwise(x, want["x"], "fixed x")


@pytest.mark.parametrize("small", [True, False])
def test_small_loop_breakdown(ctx, small):
    a = O.gen_stencil("poisson7", 6, 6, 6)
    m = 4
    b = O.rhs(a.n, m, 0)
    b[2::m] = 0.0   # column 2: zero RHS -> delta = 0 at iteration 0
    want = O.solve(a, b, m, "bicgstab", "merged", fixed=True, maxit=5)
    assert (want["breakdown"], want["breakdown_iter"], want["breakdown_col"]) == (1, 0, 2)
    with pytest.raises(P.BreakdownError, match="iteration 0, column 2"):
        run(ctx, a, b, m, "merged", small, fixed=True, max_iters=5)
