"""The reference CPU implementation (oracle/_ref: the reference's own
core::spmv + kernels::execute_group under the restated merged solvers) on the
BASELINE configs, on this box's host cores: a few fixed iterations per config
-> RHS-iterations/s, next to the GPU numbers of tools/sweep.py.

usage: python tools/cpu_reference_configs.py [--iters 3] [--configs 2,3,4,5]"""
import argparse
import json
import os
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path[:0] = [str(ROOT), str(ROOT / "tests")]
import oracle_ctypes as O  # noqa: E402
import paper_1907_12874_b200 as P  # noqa: E402

RUNS = {2: ("convdiff7", (128, 128, 128), 1, 8, "bicgstab"),
        3: ("stencil27", (192, 192, 192), 2, 16, "rbicgstab"),
        4: ("convdiff7", (320, 320, 320), 3, 32, "pipebicgstab"),
        5: ("banded", (8_000_000,), 4, 8, "bicgstab")}


def mem_gb():
    for line in open("/proc/meminfo"):
        if line.startswith("MemAvailable:"):
            return int(line.split()[1]) / 1e6
    return 0.0


ap = argparse.ArgumentParser()
ap.add_argument("--iters", type=int, default=3)
ap.add_argument("--configs", default="2,3,4,5")
args = ap.parse_args()
threads = os.cpu_count() or 1
for cid in [int(c) for c in args.configs.split(",")]:
    kind, dims, seed, m, method = RUNS[cid]
    a = P.gen_banded(dims[0], 65536, 16, 32, seed) if kind == "banded" else P.gen_stencil(kind, *dims, seed=seed)
    need = (15 * a.n_rows * m * 8 + 12 * a.nnz()) / 1e9 * 1.2   # the shim's 15 vectors + CSR
    if need > 0.8 * mem_gb():
        print(json.dumps({"config": cid, "method": method, "m": m, "cpu": "not run (RAM)", "need_GB": round(need, 1),
                          "available_GB": round(mem_gb(), 1)}), flush=True)
        continue
    b = P.gen_rhs(a.n_rows, m, seed)
    c = O.Csr(a.n_rows, a.row_offsets, a.col_indices, a.values)
    _, its, secs = O.ref_solve(c, b, m, method, fixed=True, maxit=args.iters, threads=threads, timing=True)
    print(json.dumps({"config": cid, "method": method, "m": m, "cpu_threads": threads,
                      "cpu_ms_per_iteration": round(1e3 * secs / its, 2),
                      "cpu_rhs_it_per_s": round(m * its / secs, 1), "iterations_sampled": its}), flush=True)
