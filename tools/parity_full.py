#!/usr/bin/env python
"""Full-size parity: GPU solve vs the CPU oracle at BASELINE.json sizes.

Test infrastructure (imports oracle/ as the checker).  For every case the
GPU solve (product library, stencil twin where the config is a stencil) and
the oracle (oracle/liborc.so, OpenMP on the host cores) run on the SAME
matrix and RHS (the oracle's generator output, uploaded as-is); the record
holds iterations, residual histories and solution vectors compared bit for
bit, plus the final true residual ||b - A x|| / ||b|| of both.

  C2  conv-diff 128^3 m=8, tol 1e-8: classical / Reordered / Pipelined x
      merged / fused / basic (fused rounds exactly like merged)
  C3  27-pt 192^3 m=16, tol 1e-8: Reordered fused + merged
  C5  banded n=8M, m in {1, 8, 32}, fixed 100: all three methods (fused)
  C4  conv-diff 320^3 m=32, fixed 200, Pipelined fused on the GPU; the oracle
      runs the column subset 0..3 (m=4): columns are independent bit for bit
      (per-column scalars, per-(row, column) sums, RHS keyed by (row, column))

For the fixed-iteration C5 runs it also records the true-residual trajectory
of the GPU solve (fixed runs of k iterations, k = 5 .. 100) and the first
iteration where the recursive residual reaches rounding level, so a growing
gap between recursive and true residual can be attributed.

  python tools/parity_full.py --out gpurun_out/r02_parity_full.jsonl [--cases C2,C3,C5,C4]
"""
from __future__ import annotations

import argparse
import hashlib
import json
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

import oracle_ctypes as O  # noqa: E402
import paper_1907_12874_b200 as P  # noqa: E402


def sha(a: O.Csr) -> str:
    h = hashlib.sha256()
    for arr in (a.off, a.col, a.val):
        h.update(np.ascontiguousarray(arr).tobytes())
    return h.hexdigest()[:16]


def bits_equal(x: np.ndarray, y: np.ndarray) -> bool:
    return x.shape == y.shape and np.array_equal(np.ascontiguousarray(x).view(np.int64),
                                                 np.ascontiguousarray(y).view(np.int64))


def mismatch(x: np.ndarray, y: np.ndarray) -> dict:
    if x.shape != y.shape:
        return {"shape": [list(x.shape), list(y.shape)]}
    d = np.ascontiguousarray(x).view(np.int64) != np.ascontiguousarray(y).view(np.int64)
    with np.errstate(all="ignore"):
        rel = np.abs(x - y) / np.maximum(np.abs(y), 1e-300)
    return {"count": int(d.sum()), "first": int(np.argmax(d)) if d.any() else None,
            "max_rel": float(np.nanmax(rel)) if d.any() else 0.0}


def true_res_cpu(a: O.Csr, b: np.ndarray, x: np.ndarray, m: int) -> list:
    r = b - O.spmv(a, x, m)
    r = r.reshape(-1, m)
    bb = b.reshape(-1, m)
    return [float(np.sqrt(O.dot_exact(r[:, c].copy(), r[:, c].copy(), 1)[0]) /
                  np.sqrt(O.dot_exact(bb[:, c].copy(), bb[:, c].copy(), 1)[0])) for c in range(m)]


def gen(case):
    if case["kind"] == "banded":
        return O.gen_banded(case["n"], 65536, 16, 32, case["seed"])
    return O.gen_stencil(case["kind"], *case["grid"], seed=case["seed"])


def product_gen_sha(case) -> str:
    if case["kind"] == "banded":
        a = P.gen_banded(case["n"], 65536, 16, 32, case["seed"])
    else:
        a = P.gen_stencil(case["kind"], *case["grid"], seed=case["seed"])
    return sha(O.Csr(a.n_rows, a.row_offsets, a.col_indices, a.values))


def emit(out, rec):
    print(json.dumps({k: v for k, v in rec.items() if k not in ("trajectory",)})[:400], flush=True)
    with open(out, "a") as f:
        f.write(json.dumps(rec) + "\n")


def run_case(ctx, out, name, case, runs, sub_cols=None, trajectory=False):
    t0 = time.time()
    a = gen(case)
    m = case["m"]
    b = O.rhs(a.n, m, case["seed"])
    gen_ok = product_gen_sha(case) == sha(a)
    d = ctx.upload(P.CsrMatrix(a.n, a.off, a.col, a.val))
    stencil = 0
    if case["kind"] != "banded":
        d.set_grid(*case["grid"])
        stencil = d.stencil_kind
    B = ctx.multivector(a.n, m, b)
    X = ctx.multivector(a.n, m)
    oracle_cache = {}
    print(f"[{name}] setup {time.time() - t0:.1f}s n={a.n} nnz={a.nnz} m={m} stencil={stencil}", flush=True)
    for method, form in runs:
        X.fill(0.0)
        tg = time.time()
        rep = P.solve(ctx, d, B, X, method, form, case["tol"], case["fixed"], case["maxit"], history=True)
        xg = X.download()
        tres_gpu = [float(v) for v in P.true_residual(ctx, d, B, X)]
        tg = time.time() - tg
        oform = "basic" if form == "basic" else "merged"
        key = (method, oform)
        to = time.time()
        if key not in oracle_cache:
            if sub_cols:
                bs = np.ascontiguousarray(b.reshape(-1, m)[:, :sub_cols])
                assert bits_equal(bs.reshape(-1), O.rhs(a.n, sub_cols, case["seed"])), "RHS not column-keyed"
                want = O.solve(a, bs.reshape(-1), sub_cols, method, oform, case["tol"], case["fixed"],
                               case["maxit"])
                want["tres"] = true_res_cpu(a, bs.reshape(-1), want["x"], sub_cols)
            else:
                want = O.solve(a, b, m, method, oform, case["tol"], case["fixed"], case["maxit"])
                want["tres"] = true_res_cpu(a, b, want["x"], m)
            oracle_cache[key] = want
        want = oracle_cache[key]
        to = time.time() - to
        if sub_cols:
            hg = np.ascontiguousarray(rep.residual_history[:, :sub_cols])
            xgc = np.ascontiguousarray(xg.reshape(-1, m)[:, :sub_cols]).reshape(-1)
            tg_cmp = tres_gpu[:sub_cols]
        else:
            hg, xgc, tg_cmp = rep.residual_history, xg, tres_gpu
        rec = {"case": name, "method": method, "formulation": form, "m": m, "rows": a.n, "nnz": a.nnz,
               "operator": f"stencil twin ({stencil}-pt)" if stencil else "CSR",
               "columns_compared": sub_cols or m, "generator_equal": gen_ok,
               "iterations_gpu": rep.iterations, "iterations_oracle": want["iterations"],
               "iterations_equal": rep.iterations == want["iterations"],
               "history_bitwise": bits_equal(hg, want["hist"]), "x_bitwise": bits_equal(xgc, want["x"]),
               "converged_gpu": rep.converged, "breakdown_gpu": rep.breakdown,
               "true_residual_gpu_max": max(tg_cmp), "true_residual_oracle_max": max(want["tres"]),
               "true_residual_gpu_all_columns_max": max(tres_gpu),
               "final_recursive_residual_max": float(np.nanmax(rep.residual_history[-1])),
               "gpu_s": round(tg, 2), "oracle_s": round(to, 2)}
        rec["pass"] = bool(rec["iterations_equal"] and rec["history_bitwise"] and rec["x_bitwise"] and gen_ok)
        if not rec["history_bitwise"]:
            rec["history_mismatch"] = mismatch(hg, want["hist"]) if hg.shape == want["hist"].shape else "shape"
        if not rec["x_bitwise"]:
            rec["x_mismatch"] = mismatch(xgc, want["x"])
        h = rep.residual_history
        hmax = np.nanmax(h, axis=1)
        below = np.nonzero(hmax < 1e-14)[0]
        rec["first_iteration_recursive_below_1e-14"] = int(below[0]) if below.size else None
        rec["recursive_residual_max_at"] = {str(k): float(hmax[k]) for k in (0, 5, 10, 15, 20, 30, 40, 60, 80, 100,
                                                                             150, 200) if k < len(hmax)}
        if trajectory and case["fixed"]:
            traj = {}
            for k in (5, 10, 15, 20, 25, 30, 40, 50, 60, 80, 100):
                if k > case["maxit"]:
                    break
                X.fill(0.0)
                r2 = P.solve(ctx, d, B, X, method, form, case["tol"], True, k, history=False)
                traj[str(k)] = {"iterations": r2.iterations,
                                "true_residual_max": float(max(P.true_residual(ctx, d, B, X)))}
            rec["true_residual_trajectory"] = traj
        emit(out, rec)
    del d


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--out", default=str(ROOT / "gpurun_out" / "parity_full.jsonl"))
    p.add_argument("--cases", default="C2,C3,C5,C4")
    p.add_argument("--c5-m", default="1,8,32")
    args = p.parse_args()
    Path(args.out).parent.mkdir(parents=True, exist_ok=True)
    ctx = P.Context(0)
    ctx.set_small_path(False)
    three = ("bicgstab", "rbicgstab", "pipebicgstab")
    for c in args.cases.split(","):
        if c == "C2":
            case = dict(kind="convdiff7", grid=(128, 128, 128), m=8, seed=1, tol=1e-8, maxit=1000, fixed=False)
            run_case(ctx, args.out, "C2", case, [(mt, f) for mt in three for f in ("fused", "merged", "basic")])
        elif c == "C3":
            case = dict(kind="stencil27", grid=(192, 192, 192), m=16, seed=2, tol=1e-8, maxit=1000, fixed=False)
            run_case(ctx, args.out, "C3", case, [("rbicgstab", "fused"), ("rbicgstab", "merged")])
        elif c == "C5":
            for m in [int(v) for v in args.c5_m.split(",")]:
                case = dict(kind="banded", n=8_000_000, m=m, seed=4, tol=1e-8, maxit=100, fixed=True)
                run_case(ctx, args.out, f"C5m{m}", case, [(mt, "fused") for mt in three], trajectory=True)
        elif c == "C4":
            case = dict(kind="convdiff7", grid=(320, 320, 320), m=32, seed=3, tol=1e-8, maxit=200, fixed=True)
            run_case(ctx, args.out, "C4", case, [("pipebicgstab", "fused")], sub_cols=4)
    ctx.close()


if __name__ == "__main__":
    main()
