"""Where does the one-launch small path (small.cu) stop paying?  Times the
classical fused solve with the small path on and off over growing Poisson
grids (m = 1 and 8); prints ms/iteration for both.

usage: python tools/small_threshold.py"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_1907_12874_b200 as P  # noqa: E402

ctx = P.Context(0)
for g, m in [(32, 1), (48, 1), (64, 1), (80, 1), (100, 1), (32, 8), (40, 8), (50, 8)]:
    a = P.gen_stencil("poisson7", g, g, g)
    d = ctx.upload(a)
    B = ctx.multivector(a.n_rows, m, P.gen_rhs(a.n_rows, m, 0))
    X = ctx.multivector(a.n_rows, m)
    res = {}
    for small in (True, False):
        ctx.set_small_path(small)
        best = None
        for _ in range(3):
            X.fill(0.0)
            rep = P.solve(ctx, d, B, X, "bicgstab", "fused", fixed=True, max_iters=50, history=False)
            best = rep.loop_ms if best is None else min(best, rep.loop_ms)
        res[small] = best / 50
    ctx.set_small_path(True)
    print(f"poisson {g}^3 m={m} len={a.n_rows * m:>9}: small {res[True]:.4f} ms/it, multi-kernel {res[False]:.4f} ms/it")
