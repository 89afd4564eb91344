"""Run a few iterations of one BASELINE config solve (for ncu / nsight capture).

usage: python tools/profile_solve.py [--config 2] [--method bicgstab] [--iters 4]
"""
import argparse
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import paper_1907_12874_b200 as P  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--grid", type=int, default=128)
ap.add_argument("--kind", default="convdiff7")
ap.add_argument("--m", type=int, default=8)
ap.add_argument("--method", default="bicgstab")
ap.add_argument("--formulation", default="merged")
ap.add_argument("--iters", type=int, default=4)
ap.add_argument("--seed", type=int, default=1)
ap.add_argument("--hint", action="store_true", help="declare the grid (stencil twin)")
args = ap.parse_args()

g = args.grid
a = P.gen_stencil(args.kind, g, g, g, seed=args.seed) if args.kind != "banded" else P.gen_banded(8_000_000)
b = P.gen_rhs(a.n_rows, args.m, args.seed)
ctx = P.Context(0)
d = ctx.upload(a)
if args.hint and args.kind != "banded":
    d.set_grid(g, g, g)
B = ctx.multivector(a.n_rows, args.m, b)
X = ctx.multivector(a.n_rows, args.m)
rep = P.solve(ctx, d, B, X, args.method, args.formulation, fixed=True, max_iters=args.iters)
print("iterations", rep.iterations, "launches", rep.gpu_launches, "loop_ms", rep.loop_ms)
