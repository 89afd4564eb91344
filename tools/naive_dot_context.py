"""SURVEY.md 8(c) context: the UNMODIFIED reference kernels (thread-blocked
naive dots, execute.cpp:141-157) at several thread counts against the exact-dot
oracle (= the GPU path, bitwise): iteration counts and how fast the relative
residual histories drift apart.  CPU only (oracle/_ref).

usage: python tools/naive_dot_context.py [--out profiles/r01m_naive_dot_context.md]"""
import argparse
import os
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path[:0] = [str(ROOT), str(ROOT / "tests")]
import numpy as np  # noqa: E402
import oracle_ctypes as O  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--out", default=str(ROOT / "profiles" / "r01m_naive_dot_context.md"))
args = ap.parse_args()

cases = [("C1 Poisson 32^3, m=1, seed 0", O.gen_stencil("poisson7", 32, 32, 32), 1, 0),
         ("conv-diff 48^3, m=4, seed 1", O.gen_stencil("convdiff7", 48, 48, 48, seed=1), 4, 1)]
threads = [t for t in (1, 2, 4, 8, 16) if t <= (os.cpu_count() or 1)]
lines = ["# r01m -- exact dots vs the reference's naive dots (SURVEY.md 8(c) context)", "",
         "The exact oracle (bitwise = the GPU path at any GPU count) against the reference's own kernels",
         "(`oracle/_ref`: core::spmv + kernels::execute_group, naive thread-blocked dots) at several thread",
         "counts.  Max relative history difference at iterations 5 / 10 / 15 / 20 / 30, and iterations to",
         "tol 1e-8.  The reference does not agree with itself across thread counts either.", ""]
for method in ("bicgstab", "rbicgstab", "pipebicgstab"):
    for name, a, m, seed in cases:
        b = O.rhs(a.n, m, seed)
        ex = O.solve(a, b, m, method, "merged", 1e-8)
        lines += [f"## {method}, {name}", "",
                  "| dots | iterations | hist diff @5 | @10 | @15 | @20 | @30 |", "|---|---|---|---|---|---|---|",
                  f"| exact (oracle = GPU) | {ex['iterations']} | 0 | 0 | 0 | 0 | 0 |"]
        for t in threads:
            _, its, h = O.ref_solve_hist(a, b, m, method, 1e-8, threads=t)
            cells = []
            for j in (5, 10, 15, 20, 30):
                if j < len(h) and j < len(ex["hist"]):
                    cells.append(f"{np.max(np.abs(h[j] - ex['hist'][j]) / ex['hist'][j]):.1e}")
                else:
                    cells.append("-")
            lines.append(f"| naive, {t} thread{'s' if t > 1 else ''} | {its} | " + " | ".join(cells) + " |")
        lines.append("")
Path(args.out).write_text("\n".join(lines) + "\n")
print("\n".join(lines))
