"""The paper's own benchmark (Tab. 'loop_exec_time_nv'): 7-point Poisson on
a 200^3 grid (8M unknowns), fixed 1000 iterations, six methods, basic and merged
formulations, m = 1, 4, 16 -- per-iteration times on one B200 next to the published
Lomonosov-2 node times.

usage: python tools/paper_table.py [--iters 1000] [--out profiles/r01r_paper_table.md]"""
import argparse
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import paper_1907_12874_b200 as P  # noqa: E402

# PAPER.md:470-484 (Lomonosov-2 node, seconds per iteration): (basic, merged) for m = 1, 4, 16
PUBLISHED = {
    "bicgstab": ((0.062, 0.058), (0.181, 0.164), (0.65, 0.59)),
    "ibicgstab": ((0.074, 0.061), (0.236, 0.182), (0.87, 0.66)),
    "pipebicgstab": ((0.087, 0.069), (0.282, 0.212), (1.06, 0.78)),
    "pbicgstab": ((0.066, 0.064), (0.201, 0.189), (0.72, 0.68)),
    "rbicgstab": ((0.072, 0.065), (0.224, 0.196), (0.81, 0.7)),
    "ppipebicgstab": ((0.107, 0.085), (0.368, 0.279), (1.39, 1.03)),
}
ap = argparse.ArgumentParser()
ap.add_argument("--iters", type=int, default=1000)
ap.add_argument("--out", default=str(ROOT / "profiles" / "r01r_paper_table.md"))
args = ap.parse_args()
ctx = P.Context(0)
g = 200
a = P.gen_poisson_7pt(g, g, g)
d = ctx.upload(a)
d.set_grid(g, g, g)
lines = ["# r01r -- the paper's benchmark on one B200", "",
         f"7-point Poisson {g}^3 (8M unknowns), fixed {args.iters} iterations, RHS u[-1,1] seed 0, one B200;",
         "milliseconds per iteration (paper: Lomonosov-2 node, PAPER.md:461-480, seconds -> ms).", "",
         "| method | m | basic (B200) | merged (B200) | fused (B200) | paper basic | paper merged | speed-up (merged) |",
         "|---|---|---|---|---|---|---|---|"]
methods = ["bicgstab", "ibicgstab", "pipebicgstab", "pbicgstab", "rbicgstab", "ppipebicgstab"]
for mi, m in enumerate((1, 4, 16)):
    B = ctx.multivector(a.n_rows, m, P.gen_rhs(a.n_rows, m, 0))
    X = ctx.multivector(a.n_rows, m)
    for meth in methods:
        t = {}
        for form in ("basic", "merged", "fused"):
            if form == "fused" and m not in (1, 2, 4, 8, 16, 32):
                continue
            best = None
            for _ in range(2):
                X.fill(0.0)
                rep = P.solve(ctx, d, B, X, meth, form, fixed=True, max_iters=args.iters, history=False)
                best = rep.loop_ms if best is None else min(best, rep.loop_ms)
            t[form] = best / args.iters
        pub = PUBLISHED.get(meth)
        pb, pm = (pub[mi][0] * 1e3, pub[mi][1] * 1e3) if pub else (None, None)
        sp = f"{pm / t['merged']:.0f}x" if pm else "-"
        lines.append(f"| {meth} | {m} | {t['basic']:.3f} | {t['merged']:.3f} | {t.get('fused', float('nan')):.3f} | "
                     f"{pb if pb else '-'} | {pm if pm else '-'} | {sp} |")
        print(lines[-1], flush=True)
    del B, X
Path(args.out).write_text("\n".join(lines) + "\n")
