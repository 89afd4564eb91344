"""GPU parity of the CSR SpMM on the length-sorted twin (spmm.cu
build_sorted_twin): rows stored by descending length inside windows so that a
warp's lanes and a tile's warps walk rows of one length.  Only the storage
order of the rows changes -- every (row, column) sum is the reference's
sequence (spmv.cpp:38-47) -- so results stay bitwise the oracle's.
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
def env(**kw):
    old = {k: os.environ.get(k) for k in kw}
    os.environ.update({k: str(v) for k, v in kw.items()})
    try:
        yield
    finally:
        for k, v in old.items():
            if v is None:
                del os.environ[k]
            else:
                os.environ[k] = v


def ragged(n, seed, long_rows=()):
    """Rows of 0..40 nonzeros plus a few very long ones (beyond one tile)."""
    rng = np.random.default_rng(seed)
    off, cols, vals = [0], [], []
    for i in range(n):
        k = dict(long_rows).get(i, int(rng.integers(0, 41)))
        c = np.sort(rng.choice(n, size=k, replace=False)).astype(np.int32)
        cols.append(c)
        vals.append(rng.standard_normal(k))
        off.append(off[-1] + k)
    return O.Csr(n, np.array(off, np.int64), np.concatenate(cols).astype(np.int32), np.concatenate(vals))


def test_sort_heuristic(ctx):
    """Stencil operators keep the natural order; the random band (config 5's
    shape: 16-32 nonzeros per row) gets the twin; the environment overrides."""
    st = ctx.upload(to_prod(O.gen_stencil("stencil27", 16, 16, 16, seed=2)))
    assert not st.sort_info()[0] and st.sort_info()[1] > 0.92
    cd = ctx.upload(to_prod(O.gen_stencil("convdiff7", 20, 20, 20)))
    assert not cd.sort_info()[0]
    band = to_prod(O.gen_banded(20_000, 4096, 16, 32, 4))
    d = ctx.upload(band)
    so, eff = d.sort_info()
    assert so and 0.7 < eff < 0.9
    with env(MBG_SPMM_SORT=0):
        assert not ctx.upload(band).sort_info()[0]
    with env(MBG_SPMM_SORT=1):
        assert ctx.upload(to_prod(O.gen_stencil("convdiff7", 20, 20, 20))).sort_info()[0]


@pytest.mark.parametrize("mname", list(MATRICES))
@pytest.mark.parametrize("m", [2, 4, 8, 16, 32])   # the twin serves m >= 4; m = 2 keeps the natural order
@pytest.mark.parametrize("window", [64, 4096])
def test_spmv_sorted_forced(ctx, mname, m, window):
    a = MATRICES[mname]()
    x = np.random.default_rng(200 + m).standard_normal(a.n * m)
    want = O.spmv(a, x, m)
    with env(MBG_SPMM_SORT=1, MBG_SPMM_SORT_WINDOW=window):
        d = ctx.upload(to_prod(a))
    assert d.sort_info()[0]
    X = ctx.multivector(a.n, m, x)
    Y = ctx.multivector(a.n, m)
    P.spmv(ctx, d, X, Y)
    assert_bitwise(Y.download(), want, f"sorted spmv {mname} m={m} window={window}")


@pytest.mark.parametrize("m", [1, 2, 3, 8, 32])
def test_spmv_sorted_ragged_long_and_empty_rows(ctx, m):
    """Empty rows, rows at the twin's longest (240 nonzeros = the 60 batches of
    a stage) and beyond it (multiplied by the long-row kernel); m = 3 takes the
    generic kernel on the original storage."""
    n = 6001                      # not a multiple of 8: the last group has padding slots
    a = ragged(n, 11, long_rows={5: 239, 6: 240, 7: 241, 700: 1920, 701: 1921, 3000: 5000, 5999: 2500})
    x = np.random.default_rng(m).standard_normal(n * m)
    with env(MBG_SPMM_SORT_WINDOW=512):
        d = ctx.upload(to_prod(a))
    assert d.sort_info()[0]
    X = ctx.multivector(n, m, x)
    Y = ctx.multivector(n, m)
    Y.fill(7.0)
    P.spmv(ctx, d, X, Y)
    assert_bitwise(Y.download(), O.spmv(a, x, m), f"ragged sorted spmv m={m}")


@pytest.mark.parametrize("m", [8, 16])
def test_solve_sorted_long_rows_fused_epilogue(ctx, m):
    """Fused SpMM epilogues (exact dots of finished rows) when some rows take
    the long-row kernel: their terms come from the epilogue-only tiles."""
    n = 3000
    rng = np.random.default_rng(3)
    off, cols, vals = [0], [], []
    for i in range(n):
        k = 400 if i in (11, 1500) else int(rng.integers(3, 12))
        c = np.unique(np.concatenate([[i], rng.choice(n, size=k - 1, replace=False)])).astype(np.int32)
        v = -rng.random(c.size)
        v[c == i] = 1.1 * (np.abs(v).sum() + 1.0)       # diagonally dominant
        cols.append(c)
        vals.append(v)
        off.append(off[-1] + c.size)
    a = O.Csr(n, np.array(off, np.int64), np.concatenate(cols), np.concatenate(vals))
    b = O.rhs(n, m, 7)
    ctx.set_small_path(False)
    try:
        with env(MBG_SPMM_SORT=1):
            d = ctx.upload(to_prod(a))
        assert d.sort_info()[0]
        for method in ("bicgstab", "rbicgstab"):
            want = O.solve(a, b, m, method, "fused", 1e-8, True, 12)
            B, X = ctx.multivector(n, m, b), ctx.multivector(n, m)
            rep = P.solve(ctx, d, B, X, method, "fused", 1e-8, True, 12)
            assert_same_solve(want, rep, X, f"long rows {method} m={m}")
    finally:
        ctx.set_small_path(True)


@pytest.mark.parametrize("form", ["merged", "basic", "fused"])
@pytest.mark.parametrize("method", ["bicgstab", "rbicgstab", "pipebicgstab"])
@pytest.mark.parametrize("m", [2, 8])
def test_solve_sorted_banded(ctx, method, form, m):
    """The fused SpMM epilogues (exact dots of finished rows) on the twin."""
    a = O.gen_banded(30_000, 2048, 16, 32, 4)
    b = O.rhs(a.n, m, 4)
    want = O.solve(a, b, m, method, form, 1e-8, True, 25)
    d = ctx.upload(to_prod(a))
    assert d.sort_info()[0]
    B = ctx.multivector(a.n, m, b)
    X = ctx.multivector(a.n, m)
    rep = P.solve(ctx, d, B, X, method, form, 1e-8, True, 25)
    assert_same_solve(want, rep, X, f"sorted banded {method}/{form} m={m}")


@pytest.mark.parametrize("method", ["ibicgstab", "ppipebicgstab"])
def test_solve_sorted_other_methods(ctx, method):
    """IBiCGStab also multiplies by A^T (its own twin)."""
    a = O.gen_banded(20_000, 1024, 16, 32, 4)
    b = O.rhs(a.n, 4, 4)
    pc = dict(precond_alpha=4) if method == "ppipebicgstab" else {}
    want = O.solve(a, b, 4, method, "merged", 1e-8, True, 20, **pc)
    d = ctx.upload(to_prod(a))
    assert d.sort_info()[0]
    B = ctx.multivector(a.n, 4, b)
    X = ctx.multivector(a.n, 4)
    rep = P.solve(ctx, d, B, X, method, "merged", 1e-8, True, 20, **pc)
    assert_same_solve(want, rep, X, f"sorted banded {method}")


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("method", ["bicgstab", "pipebicgstab"])
def test_sorted_partitioned_banded(ctx, world, method):
    """Interior / boundary twins of a row-block partition (emulated communicator)."""
    n, m = 24_000, 8
    a = O.gen_banded(n, 1500, 16, 32, 4)
    b = O.rhs(n, m, 4)
    bounds = [p * (n // world) for p in range(world)] + [n]
    want = O.solve(a, b, m, method, "fused", 1e-8, True, 20)
    parts = run_partitioned(a, b, m, bounds, method, "fused", tol=1e-8, fixed=True, max_iters=20)
    for r, (rep, x) in enumerate(parts):
        assert rep.iterations == want["iterations"]
        assert np.array_equal(rep.residual_history.view(np.int64), want["hist"].view(np.int64))
        r0, r1 = bounds[r], bounds[r + 1]
        assert np.array_equal(x.view(np.int64), want["x"][r0 * m:r1 * m].view(np.int64))
