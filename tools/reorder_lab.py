"""Does a brick ordering of a 3-D stencil speed up the gather-bound SpMM?

Builds P A P^T for a bx x by x bz brick ordering of the nx x ny x nz grid
(each row keeps its nonzeros in their original order, so the SpMM sums are
bitwise the unpermuted ones, and the exact-dot solver iterates identically),
then times fixed-iteration solves on both.

usage: python tools/reorder_lab.py --kind stencil27 --grid 192 --m 16 --brick 4,4,4 [--method rbicgstab]"""
import argparse
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_1907_12874_b200 as P  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--kind", default="stencil27")
ap.add_argument("--grid", type=int, default=192)
ap.add_argument("--m", type=int, default=16)
ap.add_argument("--brick", default="4,4,4")
ap.add_argument("--method", default="rbicgstab")
ap.add_argument("--formulation", default="fused")
ap.add_argument("--iters", type=int, default=40)
ap.add_argument("--seed", type=int, default=2)
args = ap.parse_args()
g = args.grid
a = P.gen_stencil(args.kind, g, g, g, seed=args.seed)
n = a.n_rows
bx, by, bz = map(int, args.brick.split(","))
# new position of row i: bricks in (z, y, x) order, lexicographic inside a brick
i = np.arange(n, dtype=np.int64)
x, y, z = i % g, (i // g) % g, i // (g * g)
nbx, nby = (g + bx - 1) // bx, (g + by - 1) // by
brick = ((z // bz) * nby + (y // by)) * nbx + (x // bx)
inner = ((z % bz) * by + (y % by)) * bx + (x % bx)
key = brick * (bx * by * bz) + inner
order = np.argsort(key, kind="stable")          # order[new] = old
pos = np.empty(n, np.int64)
pos[order] = np.arange(n)                       # pos[old] = new
t0 = time.time()
cnt = np.diff(a.row_offsets)[order]
off = np.zeros(n + 1, np.int64)
np.cumsum(cnt, out=off[1:])
# vectorised gather of each row's nonzero range
starts = a.row_offsets[order]
idx = np.repeat(starts - off[:-1], cnt) + np.arange(off[-1])
col = pos[a.col_indices[idx]].astype(np.int32)
val = a.values[idx]
ap_ = P.CsrMatrix(n, off, col, val)
print(f"permuted in {time.time() - t0:.1f}s")
m = args.m
b = P.gen_rhs(n, m, args.seed)
bp = np.ascontiguousarray(b.reshape(n, m)[order].reshape(-1))
ctx = P.Context(0)
res = {}
for name, mat, rhs in (("natural", a, b), (f"brick {args.brick}", ap_, bp)):
    d = ctx.upload(mat, any_order=True)
    B = ctx.multivector(n, m, rhs)
    X = ctx.multivector(n, m)
    best = None
    for _ in range(3):
        X.fill(0.0)
        rep = P.solve(ctx, d, B, X, args.method, args.formulation, fixed=True, max_iters=args.iters)
        best = rep.loop_ms if best is None else min(best, rep.loop_ms)
    X.fill(0.0)
    _, prof = P.solve_profile(ctx, d, B, X, args.method, args.formulation, fixed=True, max_iters=10)
    print("   ", {k: round(v[1] / v[0], 4) for k, v in prof.items()})
    X.fill(0.0)
    rep = P.solve(ctx, d, B, X, args.method, args.formulation, fixed=True, max_iters=args.iters)
    xs = X.download().reshape(n, m)
    res[name] = (best / args.iters, rep.residual_history.copy(), xs if name == "natural" else xs[pos])
    print(f"{name:16s} {best / args.iters:.4f} ms/iteration")
h0, h1 = res["natural"][1], res[f"brick {args.brick}"][1]
print("histories bitwise equal:", np.array_equal(h0.view(np.int64), h1.view(np.int64)),
      "| x bitwise equal:", np.array_equal(res["natural"][2].view(np.int64), res[f"brick {args.brick}"][2].view(np.int64)))
