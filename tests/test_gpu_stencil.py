"""GPU parity of the stencil SpMM (stencil.cu): operators declared on a grid
(mbg_csr_set_grid) run with implicit columns and TMA-staged x planes; the
result must be bit for bit the CSR oracle's (spmv.cpp:40-46 arithmetic), for
full stencils, stencils with absent entries, partial tiles, special values,
and whole solves."""
import numpy as np
import pytest

import oracle_ctypes as O
import paper_1907_12874_b200 as P
from test_gpu_parity import assert_bitwise, to_prod

pytestmark = pytest.mark.gpu

GRIDS = {
    # odd sizes: partial 32 x 4 tiles, short z ranges
    "poisson7_37x19x11": ("poisson7", (37, 19, 11), 0),
    "convdiff7_64x8x5": ("convdiff7", (64, 8, 5), 1),
    "stencil27_33x10x7": ("stencil27", (33, 10, 7), 2),
    "stencil27_3x3x3": ("stencil27", (3, 3, 3), 2),
    "convdiff7_1x1x40": ("convdiff7", (1, 1, 40), 1),
    "poisson5_45x23x1": ("poisson5", (45, 23, 1), 0),   # 2-D 5-point: one plane
}


def grid_matrix(name):
    kind, dims, seed = GRIDS[name]
    return O.gen_stencil(kind, *dims, seed=seed), dims, (27 if kind == "stencil27" else 7)


@pytest.mark.parametrize("name", list(GRIDS))
@pytest.mark.parametrize("m", [4, 8, 16, 32])
def test_stencil_spmv_bitwise(ctx, name, m):
    a, dims, kind = grid_matrix(name)
    d = ctx.upload(to_prod(a))
    d.set_grid(*dims)
    assert d.stencil_kind == kind
    x = np.random.default_rng(m).standard_normal(a.n * m)
    X, Y = ctx.multivector(a.n, m, x), ctx.multivector(a.n, m)
    P.spmv(ctx, d, X, Y)
    assert_bitwise(Y.download(), O.spmv(a, x, m), f"stencil spmv {name} m={m}")


def drop_entries(a: O.Csr, every: int) -> O.Csr:
    """Remove every `every`-th off-diagonal nonzero (absent slots inside the grid)."""
    off, cols, vals = [0], [], []
    k = 0
    for i in range(a.n):
        for q in range(a.off[i], a.off[i + 1]):
            k += 1
            if a.col[q] != i and k % every == 0:
                continue
            cols.append(a.col[q])
            vals.append(a.val[q])
        off.append(len(cols))
    return O.Csr(a.n, np.array(off), np.array(cols, np.int32), np.array(vals))


@pytest.mark.parametrize("kind,dims", [("stencil27", (40, 9, 6)), ("convdiff7", (40, 9, 6))])
def test_stencil_absent_slots(ctx, kind, dims):
    a = drop_entries(O.gen_stencil(kind, *dims, seed=3), 5)
    d = ctx.upload(to_prod(a))
    d.set_grid(*dims)
    assert d.stencil_kind in (7, 27)
    for m in (4, 8, 16, 32):
        x = np.random.default_rng(11).standard_normal(a.n * m)
        X, Y = ctx.multivector(a.n, m, x), ctx.multivector(a.n, m)
        P.spmv(ctx, d, X, Y)
        assert_bitwise(Y.download(), O.spmv(a, x, m), f"absent slots {kind} m={m}")


def test_stencil_special_values(ctx):
    # -0.0 sums, infinities and NaNs must propagate exactly as in CSR order
    a = O.gen_stencil("stencil27", 34, 6, 5, seed=2)
    m = 8
    x = np.random.default_rng(5).standard_normal(a.n * m)
    x[::97] = -0.0
    x[5 * m + 3] = np.inf
    x[77 * m + 1] = -np.inf
    x[301 * m + 6] = np.nan
    x[900 * m:901 * m] = 1e308
    d = ctx.upload(to_prod(a))
    d.set_grid(34, 6, 5)
    X, Y = ctx.multivector(a.n, m, x), ctx.multivector(a.n, m)
    P.spmv(ctx, d, X, Y)
    got, want = Y.download(), O.spmv(a, x, m)
    nan = np.isnan(want)
    assert np.array_equal(np.isnan(got), nan)
    assert_bitwise(got[~nan], want[~nan], "special values")


def test_stencil_rejects_non_grid(ctx):
    a = O.gen_banded(4096, 200, 4, 8, 4)
    d = ctx.upload(to_prod(a))
    d.set_grid(16, 16, 16)
    assert d.stencil_kind == 0
    # a 7-point operator declared on the wrong grid is no stencil either
    b = O.gen_stencil("poisson7", 8, 8, 8)
    e = ctx.upload(to_prod(b))
    e.set_grid(16, 4, 8)
    assert e.stencil_kind == 0
    m = 8
    x = np.random.default_rng(1).standard_normal(b.n * m)
    X, Y = ctx.multivector(b.n, m, x), ctx.multivector(b.n, m)
    P.spmv(ctx, e, X, Y)
    assert_bitwise(Y.download(), O.spmv(b, x, m), "wrong grid -> CSR path")


@pytest.mark.parametrize("method,form", [("bicgstab", "fused"), ("rbicgstab", "fused"), ("pipebicgstab", "merged"),
                                         ("pbicgstab", "fused"), ("ibicgstab", "merged")])
@pytest.mark.parametrize("kind,dims,m", [("convdiff7", (36, 9, 8), 8), ("stencil27", (20, 12, 9), 16),
                                         ("convdiff7", (33, 5, 6), 32), ("stencil27", (37, 17, 7), 4),
                                         ("stencil27", (35, 9, 11), 32)])
def test_stencil_solve_bitwise(ctx, method, form, kind, dims, m):
    a = O.gen_stencil(kind, *dims, seed=2)
    b = O.rhs(a.n, m, 3)
    want = O.solve(a, b, m, method, form, 1e-8, maxit=400)
    d = ctx.upload(to_prod(a))
    d.set_grid(*dims)
    assert d.stencil_kind in (7, 27)
    B, X = ctx.multivector(a.n, m, b), ctx.multivector(a.n, m)
    rep = P.solve(ctx, d, B, X, method, form, 1e-8, max_iters=400)
    assert rep.iterations == want["iterations"]
    assert_bitwise(rep.residual_history, want["hist"], f"{method} history")
    assert_bitwise(X.download(), want["x"], f"{method} x")


EPI_SCRIPT = r"""
import sys
sys.path.insert(0, {root!r}); sys.path.insert(0, {tests!r})
import test_gpu_stencil as T, paper_1907_12874_b200 as P
c = P.Context(0)
for method in ("bicgstab", "rbicgstab"):
    T.check_fused_multistep(c, method)
print("ok")
"""


def test_stencil_fused_epilogues_opt_in():
    # MBG_STENCIL_EPI=1 (read once per process): the dot epilogues of the
    # stencil SpMM, bitwise vs the oracle over many planes per block
    import os
    import subprocess
    import sys
    from pathlib import Path
    here = Path(__file__).resolve().parent
    code = EPI_SCRIPT.format(root=str(here.parent), tests=str(here))
    r = subprocess.run([sys.executable, "-c", code], env={**os.environ, "MBG_STENCIL_EPI": "1"},
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and "ok" in r.stdout, r.stdout + r.stderr


@pytest.mark.parametrize("method", ["bicgstab", "rbicgstab"])
def test_stencil_fused_epilogue_multistep(ctx, method):
    check_fused_multistep(ctx, method)


def check_fused_multistep(ctx, method):
    # enough planes per block that warps drift apart (fused dot epilogues and
    # the end-of-kernel combine must not race the last steps)
    kind, dims, m = "convdiff7", (64, 64, 48), 8
    a = O.gen_stencil(kind, *dims, seed=1)
    b = O.rhs(a.n, m, 1)
    want = O.solve(a, b, m, method, "fused", 1e-8, fixed=True, maxit=6)
    d = ctx.upload(to_prod(a))
    d.set_grid(*dims)
    B, X = ctx.multivector(a.n, m, b), ctx.multivector(a.n, m)
    rep = P.solve(ctx, d, B, X, method, "fused", 1e-8, fixed=True, max_iters=6)
    assert_bitwise(rep.residual_history, want["hist"], f"{method} fused history")
    assert_bitwise(X.download(), want["x"], f"{method} fused x")


def test_stencil_random_shapes(ctx):
    # randomized grid shapes (partial tiles in x and y, 1..20 planes) for every
    # supported m: the twin's work split (whole tiles or z-segments per block),
    # tile padding and halo zero fill against the CSR oracle
    rng = np.random.default_rng(2024)
    for _ in range(24):
        kind = ["poisson7", "convdiff7", "stencil27"][int(rng.integers(3))]
        nx, ny, nz = int(rng.integers(1, 70)), int(rng.integers(1, 19)), int(rng.integers(1, 21))
        m = [4, 8, 16, 32][int(rng.integers(4))]
        a = O.gen_stencil(kind, nx, ny, nz, seed=int(rng.integers(100)))
        d = ctx.upload(to_prod(a))
        d.set_grid(nx, ny, nz)
        assert d.stencil_kind in (7, 27)
        x = rng.standard_normal(a.n * m)
        X, Y = ctx.multivector(a.n, m, x), ctx.multivector(a.n, m)
        P.spmv(ctx, d, X, Y)
        assert_bitwise(Y.download(), O.spmv(a, x, m), f"{kind} {nx}x{ny}x{nz} m={m}")


@pytest.mark.parametrize("mode", ["0", "1", "2", "6", "epi"])
def test_stencil_z27_modes(mode):
    # the 27-point m = 16 / 32 SpMM has three implementations selected once per
    # process by MBG_STENCIL_Z (0: three resident planes; else z-marching with
    # ring depths 1: 3/2, 2: 2/2 at 2 blocks/SM, 3 (default): 4/3, 6: 5/3):
    # rerun the stencil parity tests under the non-default ones
    import os
    import subprocess
    import sys
    from pathlib import Path
    if os.environ.get("MBG_Z_NESTED"):
        pytest.skip("nested run")
    here = Path(__file__).resolve()
    # "epi": the default kernel with the opt-in delta epilogue (MBG_Z27_EPI=1)
    env = {**os.environ, "MBG_Z_NESTED": "1"}
    env.update({"MBG_Z27_EPI": "1"} if mode == "epi" else {"MBG_STENCIL_Z": mode})
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-m", "gpu", "-p", "no:cacheprovider", str(here),
                        "-k", "spmv_bitwise or absent_slots or special_values or solve_bitwise or random_shapes or axpy"],
                       env=env, capture_output=True, text=True, timeout=1200, cwd=str(here.parent.parent))
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]


@pytest.mark.parametrize("m,dims", [(16, (40, 13, 24)), (32, (33, 8, 10))])
def test_reordered_fused_axpy_spmm(ctx, m, dims):
    # fused Reordered on a 27-point twin forms th = z - alpha s inside the second
    # SpMM (th never stored) and recomputes it in the x/z/vh pass: many planes
    # per block, converged solve and a fixed-iteration one, bitwise vs the oracle
    a = O.gen_stencil("stencil27", *dims, seed=2)
    b = O.rhs(a.n, m, 5)
    d = ctx.upload(to_prod(a))
    d.set_grid(*dims)
    for fixed, maxit in ((False, 400), (True, 7)):
        want = O.solve(a, b, m, "rbicgstab", "fused", 1e-8, fixed=fixed, maxit=maxit)
        B, X = ctx.multivector(a.n, m, b), ctx.multivector(a.n, m)
        rep = P.solve(ctx, d, B, X, "rbicgstab", "fused", 1e-8, fixed=fixed, max_iters=maxit)
        assert rep.iterations == want["iterations"]
        assert_bitwise(rep.residual_history, want["hist"], "history")
        assert_bitwise(X.download(), want["x"], "x")
        # byte model: delta pass 2 (or r0 read by the SpMM epilogue: 1) + (s read
        # by the SpMM) 1 + 4-dot pass 4 + x/z/vh/r pass 10 = 17 (16) vector
        # transfers, + 2 stencil SpMMs
        import os
        nvec = 16 if os.environ.get("MBG_Z27_EPI") == "1" else 17
        if os.environ.get("MBG_STENCIL_Z") == "0":   # no z-marching kernel: th has its own pass
            nvec = 19
        per_it = rep.compulsory_bytes / rep.iterations
        spmm = 16.0 * a.n * m + 8.0 * a.nnz + 4.0 * (a.n + 1)
        assert abs(per_it - (nvec * 8.0 * a.n * m + 2 * spmm)) < 16.0, per_it
