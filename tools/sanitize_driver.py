#!/usr/bin/env python
"""Small-size driver for compute-sanitizer (memcheck / racecheck / synccheck):
every hot kernel once on tiny inputs, results checked against the oracle so a
sanitizer run also proves the instrumented launches computed the right bits.

  spmm_tma_kernel        CSR SpMM, banded matrix, m = 1, 8, 32 (+ long rows)
  stencil_spmm_kernel    7-point m = 8 and 27-point m = 4 / 16 (three-plane kernel)
  stencil27z_kernel      27-point m = 16 / 32 (MBG_STENCIL_Z, set by the caller)
  group_kernel<...>      classical fused / Reordered fused / Pipelined merged solves
  scalar_kernel          (inside the solves)
  small_classical_kernel C1-shaped one-launch solve
  generic_group_kernel   mbg_execute_group interpreter

usage: compute-sanitizer --tool memcheck python tools/sanitize_driver.py
Test infrastructure (imports oracle/)."""
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

import oracle_ctypes as O  # noqa: E402
import paper_1907_12874_b200 as P  # noqa: E402


def same(a, b, what):
    if not np.array_equal(np.ascontiguousarray(a).view(np.int64), np.ascontiguousarray(b).view(np.int64)):
        raise SystemExit(f"MISMATCH {what}")


def prod(a):
    return P.CsrMatrix(a.n, a.off, a.col, a.val)


def main():
    ctx = P.Context(0)
    # CSR SpMM
    a = O.gen_banded(3000, 300, 16, 32, 4)
    d = ctx.upload(prod(a))
    for m in (1, 8, 32):
        x = O.rhs(a.n, m, 1)
        X, Y = ctx.multivector(a.n, m, x), ctx.multivector(a.n, m)
        P.spmv(ctx, d, X, Y)
        same(Y.download(), O.spmv(a, x, m), f"csr spmm m={m}")
    # stencil SpMMs
    for kind, dims, m in (("convdiff7", (40, 9, 5), 8), ("stencil27", (37, 9, 4), 4), ("stencil27", (35, 10, 5), 16),
                          ("stencil27", (33, 6, 4), 32)):
        s = O.gen_stencil(kind, *dims, seed=2)
        ds = ctx.upload(prod(s))
        ds.set_grid(*dims)
        x = O.rhs(s.n, m, 1)
        X, Y = ctx.multivector(s.n, m, x), ctx.multivector(s.n, m)
        P.spmv(ctx, ds, X, Y)
        same(Y.download(), O.spmv(s, x, m), f"stencil {kind} m={m}")
    # solves (group + scalar kernels), multi-kernel path
    ctx.set_small_path(False)
    s = O.gen_stencil("convdiff7", 20, 12, 6, seed=1)
    for method, form, m, grid in (("bicgstab", "fused", 8, True), ("rbicgstab", "fused", 16, False),
                                  ("pipebicgstab", "merged", 4, False), ("ibicgstab", "merged", 2, False)):
        ds = ctx.upload(prod(s))
        if grid:
            ds.set_grid(20, 12, 6)
        b = O.rhs(s.n, m, 1)
        B, X = ctx.multivector(s.n, m, b), ctx.multivector(s.n, m)
        rep = P.solve(ctx, ds, B, X, method, form, 1e-8, True, 4)
        want = O.solve(s, b, m, method, form, 1e-8, True, 4)
        same(rep.residual_history, want["hist"], f"{method} {form} history")
        same(X.download(), want["x"], f"{method} {form} x")
    # one-launch small path
    ctx.set_small_path(True)
    c1 = O.gen_stencil("poisson7", 12, 12, 12)
    b = O.rhs(c1.n, 4, 0)
    dc = ctx.upload(prod(c1))
    B, X = ctx.multivector(c1.n, 4, b), ctx.multivector(c1.n, 4)
    rep = P.solve(ctx, dc, B, X, "bicgstab", "merged", 1e-8)
    want = O.solve(c1, b, 4, "bicgstab", "merged", 1e-8)
    same(rep.residual_history, want["hist"], "small path history")
    # execute_group interpreter: x = 1*x + a*p ; rho = (x, p)
    m = 3
    xv, pv = O.rhs(500, m, 5), O.rhs(500, m, 6)
    Xg, Pg = ctx.multivector(500, m, xv), ctx.multivector(500, m, pv)
    g = [P.UpdateStatement(0, [(np.ones(m), 0), (np.full(m, 0.5), 1)]), P.DotStatement(0, 1, 0)]
    P.execute_group(ctx, g, [Xg, Pg])
    ctx.close()
    print("sanitize driver ok")


if __name__ == "__main__":
    main()
