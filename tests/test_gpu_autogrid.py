"""Structured-grid detection at upload (api.cu infer_grid / detect_grid): the
reference's own calls -- CsrMatrix, core::spmv, solve, no grid argument --
reach the stencil twin for lexicographic 7- and 27-point operators; anything
else keeps the CSR kernels.  Results are bitwise the oracle's either way."""
import contextlib
import os

import numpy as np
import pytest

import oracle_ctypes as O
import paper_1907_12874_b200 as P
from test_gpu_multirank_local import run_partitioned
from test_gpu_parity import assert_bitwise, assert_same_solve, to_prod

pytestmark = pytest.mark.gpu


@contextlib.contextmanager
def autogrid(on=True):
    old = os.environ.get("MBG_AUTO_GRID")
    os.environ["MBG_AUTO_GRID"] = "1" if on else "0"
    try:
        yield
    finally:
        if old is None:
            del os.environ["MBG_AUTO_GRID"]
        else:
            os.environ["MBG_AUTO_GRID"] = old


@pytest.mark.parametrize("kind,dims,want", [("poisson7", (16, 16, 16), 7), ("convdiff7", (24, 20, 9), 7),
                                            ("convdiff7", (3, 5, 4), 7), ("stencil27", (13, 11, 10), 27),
                                            ("stencil27", (3, 3, 3), 27), ("stencil27", (40, 3, 7), 27)])
@pytest.mark.parametrize("m", [4, 8, 16, 32])
def test_detected_and_bitwise(ctx, kind, dims, want, m):
    a = O.gen_stencil(kind, *dims, seed=2)
    with autogrid():
        d = ctx.upload(to_prod(a))
    assert d.stencil_kind == want
    x = np.random.default_rng(m).standard_normal(a.n * m)
    X, Y = ctx.multivector(a.n, m, x), ctx.multivector(a.n, m)
    P.spmv(ctx, d, X, Y)
    assert_bitwise(Y.download(), O.spmv(a, x, m), f"auto stencil {kind} {dims} m={m}")
    d.clear_grid()
    assert d.stencil_kind == 0
    Y.fill(3.0)
    P.spmv(ctx, d, X, Y)
    assert_bitwise(Y.download(), O.spmv(a, x, m), f"cleared {kind} {dims} m={m}")


def test_off_by_environment(ctx):
    a = to_prod(O.gen_stencil("convdiff7", 12, 12, 12))
    with autogrid(False):
        assert ctx.upload(a).stencil_kind == 0


def perturbed(a, which):
    """A grid operator with one structural defect."""
    off, col, val = a.off.copy(), a.col.copy(), a.val.copy()
    n = a.n
    if which == "far_column":      # one interior nonzero moved off the stencil
        r = n // 2 + 3               # (an interior point of the 10 x 9 x 8 grid)
        col[off[r]] -= 2             # the row's first column: two points further left, no neighbour
    elif which == "extra_nonzero":  # one row longer than any stencil row
        r = n // 2
        have = set(col[off[r]:off[r + 1]].tolist())
        c = next(c for c in range(n) if c not in have)
        ins = int(off[r] + np.searchsorted(col[off[r]:off[r + 1]], c))
        col = np.insert(col, ins, c).astype(np.int32)
        val = np.insert(val, ins, 0.25)
        off[r + 1:] += 1
    return O.Csr(n, off, col, val)


@pytest.mark.parametrize("which", ["far_column", "extra_nonzero"])
@pytest.mark.parametrize("kind", ["convdiff7", "stencil27"])
def test_near_stencils_keep_csr(ctx, kind, which):
    a = perturbed(O.gen_stencil(kind, 10, 9, 8, seed=2), which)
    with autogrid():
        d = ctx.upload(to_prod(a))
    assert d.stencil_kind == 0
    m = 8
    x = np.random.default_rng(1).standard_normal(a.n * m)
    X, Y = ctx.multivector(a.n, m, x), ctx.multivector(a.n, m)
    P.spmv(ctx, d, X, Y)
    assert_bitwise(Y.download(), O.spmv(a, x, m), f"{kind} {which}")


def test_banded_and_tiny_keep_csr(ctx):
    with autogrid():
        assert ctx.upload(to_prod(O.gen_banded(5000, 300, 16, 32, 4))).stencil_kind == 0
        assert ctx.upload(to_prod(O.gen_stencil("poisson7", 2, 2, 2))).stencil_kind == 0   # no interior point


@pytest.mark.parametrize("method,form", [("bicgstab", "fused"), ("rbicgstab", "fused"), ("pipebicgstab", "merged")])
def test_solve_without_grid_call(ctx, method, form):
    """The reference's call sequence (upload, solve) on the multi-kernel path."""
    a = O.gen_stencil("stencil27", 18, 12, 9, seed=2)
    m = 16
    b = O.rhs(a.n, m, 2)
    want = O.solve(a, b, m, method, form, 1e-8)
    ctx.set_small_path(False)
    try:
        with autogrid():
            d = ctx.upload(to_prod(a))
        assert d.stencil_kind == 27
        B, X = ctx.multivector(a.n, m, b), ctx.multivector(a.n, m)
        rep = P.solve(ctx, d, B, X, method, form, 1e-8)
    finally:
        ctx.set_small_path(True)
    assert_same_solve(want, rep, X, f"auto grid {method}/{form}")


@pytest.mark.parametrize("world", [2, 3])
def test_partitioned_slabs_detected(ctx, world):
    """z-slabs of whole planes get the twin of their slab from the partitioned upload."""
    nx, ny, nz = 12, 10, 4 * world
    a = O.gen_stencil("convdiff7", nx, ny, nz, seed=3)
    m = 8
    b = O.rhs(a.n, m, 3)
    bounds = [p * nx * ny * 4 for p in range(world + 1)]
    want = O.solve(a, b, m, "pipebicgstab", "fused", 1e-8)
    with autogrid():
        parts = run_partitioned(a, b, m, bounds, "pipebicgstab", "fused", tol=1e-8, expect_stencil=7)
    for r, (rep, x) in enumerate(parts):
        assert rep.iterations == want["iterations"]
        assert np.array_equal(rep.residual_history.view(np.int64), want["hist"].view(np.int64))
        r0, r1 = bounds[r], bounds[r + 1]
        assert np.array_equal(x.view(np.int64), want["x"][r0 * m:r1 * m].view(np.int64))


def test_partition_across_planes_keeps_csr(ctx):
    """Row blocks that cut through a plane cannot take the slab twin: those
    ranks stay on the CSR kernels (mixed ranks give the same bits)."""
    nx, ny, nz = 10, 8, 6
    a = O.gen_stencil("convdiff7", nx, ny, nz, seed=3)
    m = 8
    b = O.rhs(a.n, m, 3)
    bounds = [0, 3 * nx * ny + 17, a.n]          # not a multiple of nx*ny
    want = O.solve(a, b, m, "bicgstab", "fused", 1e-8)
    with autogrid():
        parts = run_partitioned(a, b, m, bounds, "bicgstab", "fused", tol=1e-8, expect_stencil=0)
    for r, (rep, x) in enumerate(parts):
        assert rep.iterations == want["iterations"]
        assert np.array_equal(rep.residual_history.view(np.int64), want["hist"].view(np.int64))
        r0, r1 = bounds[r], bounds[r + 1]
        assert np.array_equal(x.view(np.int64), want["x"][r0 * m:r1 * m].view(np.int64))
