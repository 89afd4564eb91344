"""Where does the end-to-end time of one C2 solve go?  device loop (CUDA
events) vs the whole mbg_solve call (graph capture + setup) vs mbg_solve_host
(+ host<->device copies)."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402
import paper_1907_12874_b200 as P  # noqa: E402

a = P.gen_stencil("convdiff7", 128, 128, 128, seed=1)
m = 8
ctx = P.Context(0)
d = ctx.upload(a)
b = P.gen_rhs(a.n_rows, m, 1)
B = ctx.multivector(a.n_rows, m, b)
X = ctx.multivector(a.n_rows, m)
for form in ("fused",):
    for rep in range(4):
        X.fill(0.0)
        ctx.synchronize()
        t = time.perf_counter()
        r = P.solve(ctx, d, B, X, "bicgstab", form, history=False)
        t_dev = time.perf_counter() - t
        x = np.zeros(a.n_rows * m)
        t = time.perf_counter()
        r2 = P.solve_host(ctx, d, b, x, m, "bicgstab", form, history=False)
        t_host = time.perf_counter() - t
        print(f"{form}: loop {r.loop_ms:.2f} ms | mbg_solve wall {t_dev*1e3:.2f} ms | "
              f"mbg_solve_host wall {t_host*1e3:.2f} ms (its {r.iterations}/{r2.iterations})")
t = time.perf_counter()
Y = ctx.multivector(a.n_rows, m, b)
ctx.synchronize()
print(f"multivector upload 134 MB: {(time.perf_counter()-t)*1e3:.2f} ms")
