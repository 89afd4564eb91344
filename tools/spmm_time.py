"""Time the solver's SpMM alone on a BASELINE config (CUDA events via the
profile solve is overkill; this uses mbg_spmv back to back).

usage: python tools/spmm_time.py --kind convdiff7 --grid 128 --m 8 [--reps 50]"""
import argparse
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402
import paper_1907_12874_b200 as P  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--kind", default="convdiff7")
ap.add_argument("--grid", type=int, default=128)
ap.add_argument("--m", type=int, default=8)
ap.add_argument("--reps", type=int, default=50)
ap.add_argument("--seed", type=int, default=1)
ap.add_argument("--hint", action="store_true", help="declare the grid (stencil twin)")
args = ap.parse_args()
g = args.grid
a = P.gen_stencil(args.kind, g, g, g, seed=args.seed) if args.kind != "banded" else P.gen_banded(8_000_000)
ctx = P.Context(0)
d = ctx.upload(a)
if args.hint and args.kind != "banded":
    d.set_grid(g, g, g)
else:
    d.clear_grid()   # the upload detects grid operators: without --hint time the CSR kernels
m = args.m
X = ctx.multivector(a.n_rows, m, P.gen_rhs(a.n_rows, m, 1))
Y = ctx.multivector(a.n_rows, m)
for _ in range(5):
    P.spmv(ctx, d, X, Y)
ctx.synchronize()
t = time.perf_counter()
for _ in range(args.reps):
    P.spmv(ctx, d, X, Y)
ctx.synchronize()
dt = (time.perf_counter() - t) / args.reps
sk = d.stencil_kind if args.hint else 0
byt = (16.0 * a.n_rows * m + 8.0 * a.nnz() + 4.0 * a.n_rows) if sk and m in (4, 8, 16, 32) else \
    P.spmv_compulsory_bytes(a.n_rows, a.nnz(), m)
print(f"{args.kind} {g}^3 m={m} stencil={sk}: {dt*1e6:.1f} us/spmv (host-timed, includes launch), "
      f"{byt/dt/1e9:.0f} GB/s algorithmic")
