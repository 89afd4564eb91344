"""Per-kernel time breakdown of one solve (CUDA events around every launch,
mbg_solve_profile) on a BASELINE-shaped problem, with or without the
structured-grid hint.

usage: python tools/kernel_breakdown.py --kind stencil27 --grid 192 --m 16 --seed 2 --method rbicgstab
       [--formulation fused] [--iters 20] [--no-hint]"""
import argparse
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import paper_1907_12874_b200 as P  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--grid", type=int, default=128)
ap.add_argument("--kind", default="convdiff7")
ap.add_argument("--m", type=int, default=8)
ap.add_argument("--seed", type=int, default=1)
ap.add_argument("--method", default="bicgstab")
ap.add_argument("--formulation", default="fused")
ap.add_argument("--iters", type=int, default=20)
ap.add_argument("--no-hint", action="store_true")
args = ap.parse_args()
g = args.grid
a = P.gen_banded(8_000_000, 65536, 16, 32, args.seed) if args.kind == "banded" else \
    P.gen_stencil(args.kind, g, g, g, seed=args.seed)
ctx = P.Context(0)
d = ctx.upload(a)
if args.kind != "banded" and not args.no_hint:
    d.set_grid(g, g, g)
B = ctx.multivector(a.n_rows, args.m, P.gen_rhs(a.n_rows, args.m, args.seed))
X = ctx.multivector(a.n_rows, args.m)
P.solve(ctx, d, B, X, args.method, args.formulation, fixed=True, max_iters=3, history=False)   # warm-up
X.fill(0.0)
rep, prof = P.solve_profile(ctx, d, B, X, args.method, args.formulation, fixed=True, max_iters=args.iters)
tot = sum(v[1] for v in prof.values())
print(f"{args.kind} {g}^3 m={args.m} {args.method} {args.formulation} stencil={d.stencil_kind}: "
      f"{tot / args.iters:.4f} ms/iteration (profiled)")
for k, (n, ms, byt) in sorted(prof.items(), key=lambda kv: -kv[1][1]):
    gbs = byt / (ms / n / 1e3) / 1e9 if byt > 0 else 0.0
    print(f"  {k:28s} {n:5d} launches {ms / n * 1e3:9.1f} us/launch {ms / tot * 100:5.1f} %  {gbs:7.0f} GB/s")
print(json.dumps({"config": vars(args), "ms_per_iteration": tot / args.iters, "kernels": prof}))
