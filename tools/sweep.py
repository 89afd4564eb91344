"""Run the BASELINE.json configs (C1-C5) on one GPU and print one JSON line per
run: RHS-iterations/s, ms/iteration, iterations, HBM bytes/iteration and the
fraction of the measured HBM peak.  C4 (m=32, 320^3) needs ~104 GB of HBM.

usage: python tools/sweep.py [--configs 1,2,3,4,5] [--formulations merged,fused] [--reps 2]
"""
import argparse
import json
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import paper_1907_12874_b200 as P  # noqa: E402

PEAK = json.loads((ROOT / "MEASURED_PEAKS.json").read_text())["hbm_gbs"] if (ROOT / "MEASURED_PEAKS.json").exists() else 6650.0

RUNS = {
    1: [("poisson7", (32, 32, 32), 0, 1, m, dict(tol=1e-8, fixed=False, max_iters=1000))
        for m in ["bicgstab"]],
    2: [("convdiff7", (128, 128, 128), 1, 8, m, dict(tol=1e-8, fixed=False, max_iters=1000))
        for m in ["bicgstab", "rbicgstab", "pipebicgstab", "ibicgstab", "pbicgstab", "ppipebicgstab"]],
    3: [("stencil27", (192, 192, 192), 2, 16, "rbicgstab", dict(tol=1e-8, fixed=False, max_iters=1000))],
    4: [("convdiff7", (320, 320, 320), 3, 32, "pipebicgstab", dict(tol=1e-8, fixed=True, max_iters=200))],
    5: [("banded", (8_000_000,), 4, mm, meth, dict(tol=1e-8, fixed=True, max_iters=100))
        for meth in ["bicgstab", "rbicgstab", "pipebicgstab"] for mm in [1, 2, 4, 8, 16, 32]],
}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="1,2,3,4,5")
    ap.add_argument("--formulations", default="merged,fused")
    ap.add_argument("--reps", type=int, default=2)
    ap.add_argument("--natural", action="store_true", help="no structured-grid hint (no brick reordering)")
    ap.add_argument("--methods", default="", help="comma list to restrict the methods (default: all of the config)")
    args = ap.parse_args()
    ctx = P.Context(0)
    cache = {}
    for cid in [int(c) for c in args.configs.split(",")]:
        for kind, dims, seed, m, method, kw in RUNS[cid]:
            if args.methods and method not in args.methods.split(","):
                continue
            key = (kind, dims, seed)
            if key not in cache:
                cache.clear()
                t = time.time()
                a = P.gen_banded(dims[0], 65536, 16, 32, seed) if kind == "banded" else P.gen_stencil(kind, *dims, seed=seed)
                d = ctx.upload(a)
                if kind != "banded" and not args.natural:
                    d.set_grid(*dims)   # brick-reordered twin for long-row stencils (C3)
                elif args.natural:
                    d.clear_grid()      # drop the stencil twin the upload detects: CSR kernels
                cache[key] = (a, d, time.time() - t)
            a, d, tgen = cache[key]
            b = P.gen_rhs(a.n_rows, m, seed)
            B = ctx.multivector(a.n_rows, m, b)
            X = ctx.multivector(a.n_rows, m)
            for form in args.formulations.split(","):
                if form == "fused" and m not in (1, 2, 4, 8, 16, 32):
                    continue
                best = None
                for _ in range(args.reps + 1):   # first rep = warm-up
                    X.fill(0.0)
                    rep = P.solve(ctx, d, B, X, method, form, history=False, **kw)
                    if best is None or rep.loop_ms < best.loop_ms:
                        best = rep
                # the solver's own byte model (preconditioner + elided copies included)
                bi = best.compulsory_bytes / max(1, best.iterations)
                msit = best.loop_ms / max(1, best.iterations)
                print(json.dumps({
                    "config": cid, "matrix": f"{kind}{'x'.join(map(str, dims))}", "m": m, "method": method,
                    "formulation": form, "iterations": best.iterations, "converged": best.converged,
                    "ms_per_iteration": round(msit, 4), "rhs_it_per_s": round(m * best.iterations / (best.loop_ms / 1e3), 1),
                    "bytes_per_iteration": bi, "hbm_GBps": round(bi / (msit / 1e3) / 1e9, 1),
                    "hbm_frac": round(bi / (msit / 1e3) / 1e9 / PEAK, 3), "gen_upload_s": round(tgen, 1),
                    "true_res_max": float(P.true_residual(ctx, d, B, X).max())}), flush=True)
            del B, X


if __name__ == "__main__":
    main()
