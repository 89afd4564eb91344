"""GPU parity of the gather-once SpMM tiling (spmm.cu spmm_stage_kernel).

The tiling is opt-in at upload (MBG_SPMM_STAGE=1) for any matrix whose rows
fit the tile limits.  Results must be bitwise the oracle's either
way: same per-(row, column) sequential CSR-order adds, x read from shared
memory instead of L1/L2.
"""
import contextlib
import os

import numpy as np
import pytest

import oracle_ctypes as O
import paper_1907_12874_b200 as P
from test_gpu_multirank_local import run_partitioned
from test_gpu_parity import MATRICES, assert_bitwise, run_both, assert_same_solve, to_prod

pytestmark = pytest.mark.gpu


@contextlib.contextmanager
def stage(mode):
    old = os.environ.get("MBG_SPMM_STAGE")
    os.environ["MBG_SPMM_STAGE"] = str(mode)
    try:
        yield
    finally:
        if old is None:
            del os.environ["MBG_SPMM_STAGE"]
        else:
            os.environ["MBG_SPMM_STAGE"] = old


@pytest.mark.parametrize("mname", list(MATRICES))
@pytest.mark.parametrize("m", [1, 4, 8, 16, 32])
def test_spmv_stage_forced(ctx, mname, m):
    a = MATRICES[mname]()
    x = np.random.default_rng(100 + m).standard_normal(a.n * m)
    want = O.spmv(a, x, m)
    with stage(1):
        d = ctx.upload(to_prod(a))
    staged, reuse = d.stage_info()
    assert staged and reuse > 1.0
    X = ctx.multivector(a.n, m, x)
    Y = ctx.multivector(a.n, m)
    P.spmv(ctx, d, X, Y)
    assert_bitwise(Y.download(), want, f"staged spmv {mname} m={m}")


def test_stage_opt_in():
    """The gather-once tiling is opt-in (measured slower on B200: L1 already
    captures the stencil reuse); MBG_SPMM_STAGE=1 enables it."""
    ctx = P.Context(0)
    try:
        a = to_prod(O.gen_stencil("stencil27", 24, 24, 24, seed=2))
        assert not ctx.upload(a).stage_info()[0]
        with stage(1):
            d = ctx.upload(a)
        assert d.stage_info()[0] and d.stage_info()[1] > 2.0
    finally:
        ctx.close()


def test_stage_row_beyond_limits_falls_back(ctx):
    """A row with more distinct columns than a staged tile holds: the tiling
    is not built and the plain kernel runs."""
    n = 2000
    rng = np.random.default_rng(3)
    off, cols, vals = [0], [], []
    for i in range(n):
        k = 300 if i == 777 else 5
        c = np.sort(rng.choice(n, size=k, replace=False)).astype(np.int32)
        cols.append(c)
        vals.append(rng.standard_normal(k))
        off.append(off[-1] + k)
    a = O.Csr(n, np.array(off, np.int64), np.concatenate(cols), np.concatenate(vals))
    with stage(1):
        d = ctx.upload(to_prod(a))
    assert not d.stage_info()[0]
    m = 8
    x = rng.standard_normal(n * m)
    X = ctx.multivector(n, m, x)
    Y = ctx.multivector(n, m)
    P.spmv(ctx, d, X, Y)
    assert_bitwise(Y.download(), O.spmv(a, x, m), "fallback spmv")


@pytest.mark.parametrize("form", ["merged", "fused"])
@pytest.mark.parametrize("method", ["bicgstab", "rbicgstab", "pipebicgstab"])
def test_solve_stage_forced_convdiff_m8(ctx, method, form):
    a = O.gen_stencil("convdiff7", 30, 28, 26)
    b = O.rhs(a.n, 8, 1)
    with stage(1):
        want, rep, X = run_both(ctx, a, b, 8, method, form)
    assert_same_solve(want, rep, X, f"staged convdiff {method}/{form}")


@pytest.mark.parametrize("world", [2, 3])
def test_stage_partitioned_27pt(ctx, world):
    """Interior / boundary staged tilings under the emulated communicator."""
    nx, ny, nz = 14, 12, 5 * world
    a = O.gen_stencil("stencil27", nx, ny, nz, seed=2)
    m = 16
    b = O.rhs(a.n, m, 2)
    bounds = [p * nx * ny * 5 for p in range(world + 1)]
    want = O.solve(a, b, m, "rbicgstab", "fused")
    with stage(1):
        parts = run_partitioned(a, b, m, bounds, "rbicgstab", "fused", tol=1e-8)
    for r, (rep, x) in enumerate(parts):
        assert rep.iterations == want["iterations"]
        assert np.array_equal(rep.residual_history.view(np.int64), want["hist"].view(np.int64))
        r0, r1 = bounds[r], bounds[r + 1]
        assert np.array_equal(x.view(np.int64), want["x"][r0 * m:r1 * m].view(np.int64))
