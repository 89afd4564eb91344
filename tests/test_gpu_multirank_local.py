"""The partitioned (multi-GPU) solver path on ONE GPU: P contexts linked into
an emulated communicator, one host thread per rank.  Exercises the device halo
plan, the interior/boundary SpMM split, the int64-limb allreduce of every
reduction point and the side-stream ordering; the result must equal the
single-GPU solve bit for bit (exact dots make it independent of P)."""
import threading

import numpy as np
import pytest

import oracle_ctypes as O
import paper_1907_12874_b200 as P

pytestmark = pytest.mark.gpu


def bits(x):
    return np.ascontiguousarray(x, dtype=np.float64).view(np.int64)


def run_partitioned(a, b, m, bounds, method, form, grid=None, expect_stencil=None, **kw):
    world = len(bounds) - 1
    ctxs = [P.Context(0) for _ in range(world)]
    P.local_group(ctxs)
    A = P.CsrMatrix(a.n, a.off, a.col, a.val)
    out = [None] * world
    err = [None] * world

    def rank(r):
        try:
            d = ctxs[r].upload(A, bounds, r)
            if grid is not None:   # z-slab on the stencil twin
                d.set_grid(*grid)
                assert d.stencil_kind in (7, 27), "slab stencil twin not built"
            if expect_stencil is not None:   # detected by the partitioned upload itself
                assert d.stencil_kind == expect_stencil, d.stencil_kind
            r0, r1 = bounds[r], bounds[r + 1]
            B = ctxs[r].multivector(r1 - r0, m, b[r0 * m:r1 * m])
            X = ctxs[r].multivector(r1 - r0, m)
            rep = P.solve(ctxs[r], d, B, X, method, form, **kw)
            out[r] = (rep, X.download())
        except Exception as e:  # noqa: BLE001
            err[r] = e

    th = [threading.Thread(target=rank, args=(r,)) for r in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=600)
    assert not any(err), err
    for c in ctxs:
        c.close()
    return out


@pytest.mark.parametrize("world", [2, 3, 4])
@pytest.mark.parametrize("method,form", [("bicgstab", "merged"), ("rbicgstab", "fused"), ("pipebicgstab", "merged"),
                                         ("bicgstab", "fused"), ("pipebicgstab", "basic"), ("ibicgstab", "merged")])
def test_zslab_partition_equals_single_gpu(ctx, world, method, form):
    nx, ny, nz = 20, 18, 6 * world
    a = O.gen_stencil("convdiff7", nx, ny, nz)
    m = 8
    b = O.rhs(a.n, m, 1)
    bounds = [p * nx * ny * 6 for p in range(world + 1)]
    want = O.solve(a, b, m, method, form)
    parts = run_partitioned(a, b, m, bounds, method, form, tol=1e-8)
    for r, (rep, x) in enumerate(parts):
        assert rep.iterations == want["iterations"], (r, rep.iterations, want["iterations"])
        assert np.array_equal(bits(rep.residual_history), bits(want["hist"]))
        r0, r1 = bounds[r], bounds[r + 1]
        assert np.array_equal(bits(x), bits(want["x"][r0 * m:r1 * m]))


def test_banded_uneven_partition(ctx):
    a = O.gen_banded(60_000, 20_000, 16, 32, 4)
    m = 4
    b = O.rhs(a.n, m, 4)
    bounds = [0, 11_111, 29_000, 60_000]
    want = O.solve(a, b, m, "bicgstab", fixed=True, maxit=25)
    parts = run_partitioned(a, b, m, bounds, "bicgstab", "merged", fixed=True, max_iters=25)
    for r, (rep, x) in enumerate(parts):
        assert rep.iterations == 25
        assert np.array_equal(bits(rep.residual_history), bits(want["hist"]))
        assert np.array_equal(bits(x), bits(want["x"][bounds[r] * m:bounds[r + 1] * m]))


@pytest.mark.parametrize("world,planes", [(2, 5), (3, 1), (4, 2), (2, 1)])
@pytest.mark.parametrize("kind,m,method,form", [("convdiff7", 8, "bicgstab", "fused"),
                                                ("convdiff7", 4, "rbicgstab", "merged"),
                                                ("stencil27", 16, "rbicgstab", "fused"),
                                                ("convdiff7", 32, "pipebicgstab", "merged")])
def test_zslab_stencil_twin_equals_single_gpu(ctx, world, planes, kind, m, method, form):
    # each rank's slab runs on its stencil twin: interior planes while the halo
    # planes travel, then the two faces reading the halo through a second
    # tensor map -- bitwise the single-GPU oracle
    nx, ny, nz = 33, 9, planes * world
    a = O.gen_stencil(kind, nx, ny, nz, seed=2)
    b = O.rhs(a.n, m, 1)
    bounds = [p * nx * ny * planes for p in range(world + 1)]
    want = O.solve(a, b, m, method, form, fixed=True, maxit=12)
    parts = run_partitioned(a, b, m, bounds, method, form, grid=(nx, ny, nz), fixed=True, max_iters=12)
    for r, (rep, x) in enumerate(parts):
        assert np.array_equal(bits(rep.residual_history), bits(want["hist"])), r
        r0, r1 = bounds[r], bounds[r + 1]
        assert np.array_equal(bits(x), bits(want["x"][r0 * m:r1 * m])), r


@pytest.mark.parametrize("world", [2, 3])
def test_ibicgstab_banded_partition_transpose_halo(ctx, world):
    # f0 = A^T r0 across ranks: the random band is not structurally symmetric,
    # so A^T's halo plan differs from A's; bitwise the single-GPU oracle
    a = O.gen_banded(30_000, 5_000, 8, 16, 7)
    m = 4
    b = O.rhs(a.n, m, 2)
    bounds = [0, 9_000, 30_000] if world == 2 else [0, 7_000, 19_500, 30_000]
    want = O.solve(a, b, m, "ibicgstab", "merged", fixed=True, maxit=15)
    parts = run_partitioned(a, b, m, bounds, "ibicgstab", "merged", fixed=True, max_iters=15)
    for r, (rep, x) in enumerate(parts):
        assert np.array_equal(bits(rep.residual_history), bits(want["hist"])), r
        assert np.array_equal(bits(x), bits(want["x"][bounds[r] * m:bounds[r + 1] * m])), r


@pytest.mark.parametrize("world", [2, 3])
def test_partitioned_spmv_transpose(ctx, world):
    # core::spmv_transpose across ranks (A^T halo plan), bitwise the serial order
    a = O.gen_banded(12_000, 3_000, 6, 12, 5)
    m = 3
    x = np.random.default_rng(9).standard_normal(a.n * m)
    want = O.spmv_transpose(a, x, m)
    bounds = [a.n * p // world for p in range(world + 1)]
    ctxs = [P.Context(0) for _ in range(world)]
    P.local_group(ctxs)
    A = P.CsrMatrix(a.n, a.off, a.col, a.val)
    out, err = [None] * world, [None] * world

    def rank(r):
        try:
            d = ctxs[r].upload(A, bounds, r)
            r0, r1 = bounds[r], bounds[r + 1]
            X = ctxs[r].multivector(r1 - r0, m, x[r0 * m:r1 * m])
            Y = ctxs[r].multivector(r1 - r0, m)
            P.spmv_transpose(ctxs[r], d, X, Y)
            out[r] = Y.download()
        except Exception as e:  # noqa: BLE001
            err[r] = e

    th = [threading.Thread(target=rank, args=(r,)) for r in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=300)
    for c in ctxs:
        c.close()
    assert not any(err), err
    for r in range(world):
        assert np.array_equal(bits(out[r]), bits(want[bounds[r] * m:bounds[r + 1] * m])), r
