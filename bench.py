#!/usr/bin/env python
"""Benchmark: RHS-iterations/s of the multi-RHS BiCGStab hot path on B200.

Default workload = BASELINE.json configs[2] (config C3), the largest config
quoted at 1/2/4/8 GPUs that a 1-GPU run covers verbatim: Reordered BiCGStab
(fused formulation = the Alg. 6 merged listing with the identity-M^-1 copies
elided, bitwise-identical results), 27-point stencil on a 192^3 grid, m=16 RHS
(seed 2), rel tol 1e-8, max 1000 iterations.  One step = one full solve from
x0 = 0 to convergence.  With N GPUs the SAME system is split into z-slabs of
whole xy-planes (strong scaling; C5 in row blocks): one process per GPU,
NCCL halo exchange + one int64-limb allreduce per reduction point.
`--config C1..C5` selects another BASELINE config (C4: Pipelined, 320^3,
m=32, fixed 200 iterations -- the 8-GPU efficiency target).

  value   RHS-iterations/s of the whole system over the timed steps (device
          CUDA events, inputs resident in HBM, max over ranks)
  e2e     same metric through the C ABI with HOST buffers: b and x0 uploaded,
          x and the history downloaded inside the timed region
  roofline dominant kernel of the iteration loop (CUDA-event profile solve in
          fixed mode over exactly the solve's iterations: no post-stop launches)
  cpu_baseline  the reference's own kernels (oracle/_ref) on the host cores
  variants the other formulations (merged = paper listing, basic) and the plain
          CSR SpMM path (what a drop-in core::spmv user gets) on the same config,
          plus config C2 classical fused / merged / basic / CSR

`python bench.py --gpus N` without torchrun re-executes itself under
`python -m torch.distributed.run --nproc-per-node N` and fails loudly when the
box has fewer than N GPUs.

`--impl reference` times the reference CPU implementation (oracle/_ref: the
reference's core::spmv + kernels::execute_group driving the restated merged
solver, all host threads) on the same config; rank 0 only.  Its inputs come
from the oracle's generators, so the product library is never loaded.
"""
from __future__ import annotations

import argparse
import json
import os
import socket
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "RHS-iterations/sec"
UNIT = "RHS-it/s"

# BASELINE.json configs (SURVEY.md Appendix A pins)
CONFIGS = {
    "C1": dict(kind="poisson7", grid=(32, 32, 32), m=1, seed=0, method="bicgstab", tol=1e-8, maxit=1000,
               fixed=False, text="classical BiCGStab, 7-pt Poisson 32^3"),
    "C2": dict(kind="convdiff7", grid=(128, 128, 128), m=8, seed=1, method="bicgstab", tol=1e-8, maxit=1000,
               fixed=False, text="classical BiCGStab, conv-diff 7-pt 128^3"),
    "C3": dict(kind="stencil27", grid=(192, 192, 192), m=16, seed=2, method="rbicgstab", tol=1e-8, maxit=1000,
               fixed=False, text="Reordered BiCGStab, 27-pt 192^3"),
    "C4": dict(kind="convdiff7", grid=(320, 320, 320), m=32, seed=3, method="pipebicgstab", tol=1e-8, maxit=200,
               fixed=True, text="Pipelined BiCGStab, conv-diff 7-pt 320^3"),
    "C5": dict(kind="banded", n=8_000_000, m=8, seed=4, method="bicgstab", tol=1e-8, maxit=100, fixed=True,
               text="random banded n=8M (16-32 nnz/row, band +-65536)"),
}


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=5)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--config", default="C3", choices=sorted(CONFIGS))
    p.add_argument("--method", default=None,
                   choices=["bicgstab", "rbicgstab", "pipebicgstab", "ibicgstab", "pbicgstab", "ppipebicgstab"])
    p.add_argument("--formulation", default="fused", choices=["merged", "basic", "fused"],
                   help="fused (default): the merged listing with beyond-paper pass merges and the identity "
                        "M^-1 copies elided -- bitwise-identical results, fewer bytes")
    p.add_argument("--m", type=int, default=None)
    p.add_argument("--tol", type=float, default=None)
    p.add_argument("--maxit", type=int, default=None)
    p.add_argument("--fixed", type=int, default=None, help="fixed iteration count instead of tol")
    p.add_argument("--no-compare", action="store_true", help="skip the variants block")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--cpu-iters", type=int, default=None, help="fixed iterations per CPU sample")
    p.add_argument("--no-grid-hint", action="store_true", help="plain CSR SpMM (drop the stencil twin the upload detects)")
    return p.parse_args()


def resolve(args):
    """The run's configuration (config defaults + explicit overrides)."""
    c = dict(CONFIGS[args.config])
    if args.method:
        c["method"] = args.method
    if args.m:
        c["m"] = args.m
    if args.tol is not None:
        c["tol"] = args.tol
    if args.fixed is not None:
        c["fixed"] = args.fixed > 0
        if args.fixed > 0:
            c["maxit"] = args.fixed
    if args.maxit is not None:
        c["maxit"] = args.maxit
    c["name"] = args.config
    c["formulation"] = args.formulation
    return c


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def n_rows(cfg):
    if cfg["kind"] == "banded":
        return cfg["n"]
    nx, ny, nz = cfg["grid"]
    return nx * ny * nz


def partition(cfg, world):
    """Row bounds per rank: z-slabs of whole xy-planes (stencils), equal row blocks (banded)."""
    if cfg["kind"] == "banded":
        n = cfg["n"]
        return [n * p // world for p in range(world + 1)]
    nx, ny, nz = cfg["grid"]
    if nz < world:
        raise SystemExit(f"bench: {nz} planes cannot be split over {world} ranks")
    return [(nz * p // world) * nx * ny for p in range(world + 1)]


def workload_desc(cfg):
    mode = f"fixed {cfg['maxit']} iterations" if cfg["fixed"] else f"rel tol {cfg['tol']:g}, max {cfg['maxit']}"
    return (f"{cfg['name']}: {cfg['text']}, method {cfg['method']} ({cfg['formulation']}), m={cfg['m']} RHS "
            f"u[-1,1] seed {cfg['seed']}, x0=0, {mode}")


def config_dict(cfg, world, nnz):
    """Identical in both arms."""
    part = "row blocks" if cfg["kind"] == "banded" else "z-slabs of xy-planes"
    return {"workload": workload_desc(cfg), "config": cfg["name"], "rows": int(n_rows(cfg)), "nnz": int(nnz),
            "m": cfg["m"], "method": cfg["method"], "formulation": cfg["formulation"],
            "tol": None if cfg["fixed"] else cfg["tol"], "fixed_iterations": cfg["maxit"] if cfg["fixed"] else None,
            "parallelism": f"{part} x{world} (strong scaling: one system split over the GPUs)",
            "units": "RHS-iterations of the whole system",
            "l2": "inputs larger than L2 (whole working set >> 126 MB; no flush needed)"}


def peaks():
    f = ROOT / "MEASURED_PEAKS.json"
    if f.exists():
        d = json.loads(f.read_text())
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md)"


class Clocks:
    """nvidia-smi sampler running during the timed region."""

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self.proc = None

    def __enter__(self):
        q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def __exit__(self, *exc):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4)
                          if len(r) > 4 + i and r[4 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


# ---------------------------------------------------------------------------
# CPU legs (test infrastructure: oracle/ only)
# ---------------------------------------------------------------------------
def oracle_problem(cfg):
    """Matrix + RHS from the oracle's generators (bit-identical to the product's)."""
    sys.path.insert(0, str(ROOT / "tests"))
    import oracle_ctypes as O
    if cfg["kind"] == "banded":
        a = O.gen_banded(cfg["n"], 65536, 16, 32, cfg["seed"])
    else:
        a = O.gen_stencil(cfg["kind"], *cfg["grid"], seed=cfg["seed"])
    return a, O.rhs(a.n, cfg["m"], cfg["seed"])


def cpu_iters(cfg, args, budget_s=15.0):
    """Fixed iterations per CPU sample: ~budget_s of work on a 16-core host
    (the reference kernels sustain ~100 GB/s of the paper's Eq. (3) bytes there)."""
    if args.cpu_iters:
        return args.cpu_iters
    n, m = n_rows(cfg), cfg["m"]
    nnz = n * {"poisson7": 7, "convdiff7": 7, "stencil27": 27, "banded": 24}[cfg["kind"]]
    eq3 = 26 * 8.0 * n * m + 2 * (8.0 * m * (n + nnz) + 4.0 * (n + 3 * nnz))
    return int(max(2, min(20, round(budget_s / (eq3 / 100e9)))))


def cpu_baseline(a, b, cfg, iters, steps=1):
    """Reference kernels (oracle/_ref) on the host cores, bounded sample."""
    sys.path.insert(0, str(ROOT / "tests"))
    import oracle_ctypes as O
    threads = os.cpu_count() or 1
    m = cfg["m"]
    method = cfg["method"] if cfg["method"] in ("bicgstab", "rbicgstab", "pipebicgstab") else "bicgstab"
    vals = []
    if O.ref_available():
        for _ in range(steps):
            _, its, secs = O.ref_solve(a, b, m, method, tol=cfg["tol"], fixed=True, maxit=iters,
                                       threads=threads, timing=True)
            vals.append(m * its / secs)
        kind = "reference"
        sample = (f"same matrix and RHS, {iters} fixed iterations of the restated merged {method} on the "
                  f"reference's core::spmv + kernels::execute_group (oracle/_ref), threads={threads}, "
                  f"setup excluded")
    else:
        for _ in range(steps):
            t = time.perf_counter()
            O.solve(a, b, m, method, "merged", cfg["tol"], True, iters)
            vals.append(m * iters / (time.perf_counter() - t))
        kind = "port"
        threads = O.orc().orc_num_threads()
        sample = f"same matrix and RHS, {iters} fixed iterations of the oracle port (OpenMP {threads} threads)"
    return {"value": float(np.median(vals)), "unit": UNIT, "cores": threads, "kind": kind, "sample": sample,
            "host": host_info()}, vals


def host_info():
    """the CPU model, memory and triad bandwidth beside the baseline."""
    import ctypes as C
    sys.path.insert(0, str(ROOT / "tests"))
    import oracle_ctypes as O
    model, mem = None, None
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
        for line in open("/proc/meminfo"):
            if line.startswith("MemTotal:"):
                mem = round(int(line.split()[1]) / 1e6, 1)
                break
    except OSError:
        pass
    lib = O.orc()
    lib.orc_triad_gbs.restype = C.c_double
    lib.orc_triad_gbs.argtypes = [C.c_long, C.c_int]
    return {"cpu_model": model, "nproc": os.cpu_count(), "mem_total_GB": mem,
            "triad_GBps": round(lib.orc_triad_gbs(40_000_000, 5), 1)}


def product_lib_mapped() -> bool:
    try:
        return "libmbstab_b200" in Path("/proc/self/maps").read_text()
    except OSError:
        return False


def run_reference(args):
    world, rank, _ = dist_env()
    if rank != 0:
        return
    cfg = resolve(args)
    a, b = oracle_problem(cfg)
    iters = cpu_iters(cfg, args, budget_s=8.0)
    steps = []
    for i in range(args.warmup + args.steps):
        cb, vals = cpu_baseline(a, b, cfg, iters, steps=1)
        if i >= args.warmup:
            steps.append(vals[0])
    if product_lib_mapped():
        raise SystemExit("bench --impl reference: the product library was loaded into the reference arm")
    value = float(np.mean(steps))
    cb["value"] = value
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1000.0 * cfg["m"] * iters / value,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded counter RNG, DESIGN.md Inputs)",
        "config": config_dict(cfg, args.gpus, a.nnz),
        "step": (f"{iters} fixed iterations of the whole system (bounded sample: the CPU's RHS-iterations/s "
                 f"do not depend on the iteration count); the reference has no fused form, so it runs the "
                 f"paper's merged listing of {cfg['method']} on its own kernels with naive dots"),
        "cpu_baseline": cb,
        "product_library_loaded": False,
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# GPU arm
# ---------------------------------------------------------------------------
def build_matrix(cfg):
    import paper_1907_12874_b200 as P
    if cfg["kind"] == "banded":
        return P.gen_banded(cfg["n"], 65536, 16, 32, cfg["seed"])
    return P.gen_stencil(cfg["kind"], *cfg["grid"], seed=cfg["seed"])


def time_solves(P, ctx, d, B, X, cfg, formulation, warmup, steps, barrier=None):
    maxit = cfg["maxit"]
    reps = []
    for i in range(warmup + steps):
        X.fill(0.0)
        r = P.solve(ctx, d, B, X, cfg["method"], formulation, cfg["tol"], cfg["fixed"], maxit, history=False)
        if i >= warmup:
            reps.append(r)
    ms = sum(r.loop_ms for r in reps) / len(reps)
    its = [r.iterations for r in reps]
    return {"formulation": formulation, "ms_per_step": ms, "iterations": its,
            "value": cfg["m"] * sum(its) / (sum(r.loop_ms for r in reps) / 1000.0),
            "ms_per_iteration": ms / max(1, its[0]),
            "bytes_per_iteration": reps[0].compulsory_bytes / max(1, reps[0].iterations)}


def variants(P, ctx, a, cfg, d, B, X, peak, steps):
    """Other formulations + the CSR path on this config (1 GPU)."""
    out = {}
    for f in ("merged", "basic"):
        if f != cfg["formulation"]:
            r = time_solves(P, ctx, d, B, X, cfg, f, 1, steps)
            r["hbm_frac"] = r["bytes_per_iteration"] / (r["ms_per_iteration"] / 1000.0) / 1e9 / peak
            out[f] = r
    if d.stencil_kind:
        dc = ctx.upload(a)
        dc.clear_grid()
        r = time_solves(P, ctx, dc, B, X, cfg, cfg["formulation"], 1, steps)
        r["operator"] = "CSR kernels (the detected stencil twin dropped: mbg_csr_clear_grid)"
        r["hbm_frac"] = r["bytes_per_iteration"] / (r["ms_per_iteration"] / 1000.0) / 1e9 / peak
        out["csr_path"] = r
        del dc
    return out


def c2_block(P, ctx, peak, steps):
    """Config C2 (classical vs merged-ops BiCGStab): fused / merged / basic on
    the stencil twin and fused on the plain CSR path."""
    cfg = resolve(argparse.Namespace(config="C2", method=None, m=None, tol=None, fixed=None, maxit=None,
                                     formulation="fused"))
    a = build_matrix(cfg)
    b = P.gen_rhs(a.n_rows, cfg["m"], cfg["seed"])
    B = ctx.multivector(a.n_rows, cfg["m"], b)
    X = ctx.multivector(a.n_rows, cfg["m"])
    out = {"workload": workload_desc(cfg)}
    d = ctx.upload(a)   # the upload detects the grid operator: no grid call, as in the reference
    for f in ("fused", "merged", "basic"):
        r = time_solves(P, ctx, d, B, X, cfg, f, 1, steps)
        r["hbm_frac"] = r["bytes_per_iteration"] / (r["ms_per_iteration"] / 1000.0) / 1e9 / peak
        r["operator"] = "stencil twin (detected at upload)" if d.stencil_kind else "CSR"
        out[f] = r
    del d
    dc = ctx.upload(a)
    dc.clear_grid()
    r = time_solves(P, ctx, dc, B, X, cfg, "fused", 1, steps)
    r["hbm_frac"] = r["bytes_per_iteration"] / (r["ms_per_iteration"] / 1000.0) / 1e9 / peak
    r["operator"] = "CSR kernels (twin dropped)"
    out["fused_csr_path"] = r
    return out


def relaunch_under_torchrun(args) -> None:
    """`bench.py --gpus N` outside torchrun: one process per GPU via torch.distributed.run."""
    if args.impl == "ours":
        import torch
        ndev = torch.cuda.device_count()
        if ndev < args.gpus:
            print(f"bench: --gpus {args.gpus} requested but this box has {ndev} CUDA device(s); refusing to "
                  f"measure fewer GPUs than asked", file=sys.stderr)
            sys.exit(2)
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), str(Path(__file__).resolve())] + sys.argv[1:]
    sys.exit(subprocess.call(cmd))


def main():
    args = parse()
    world, rank, local = dist_env()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        relaunch_under_torchrun(args)
    if "WORLD_SIZE" in os.environ and world != args.gpus:
        raise SystemExit(f"bench: --gpus {args.gpus} but WORLD_SIZE={world}")
    if args.impl == "reference":
        run_reference(args)
        return
    cfg = resolve(args)
    m = cfg["m"]
    dist = None
    if world > 1:
        os.environ.setdefault("NCCL_DEBUG", "INFO")          # rank count visible in the log
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        os.environ.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")
        import torch
        import torch.distributed as dist
        if torch.cuda.device_count() <= local:
            raise SystemExit(f"bench: rank {rank} has no GPU (LOCAL_RANK={local}, "
                             f"{torch.cuda.device_count()} device(s))")
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    import paper_1907_12874_b200 as P
    a = build_matrix(cfg)
    b_full = P.gen_rhs(a.n_rows, m, cfg["seed"])
    ctx = P.Context(local)
    bounds = None
    if world > 1:
        nid = [P.comm_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(nid, src=0)
        ctx.init_comm(rank, world, nid[0])
        bounds = partition(cfg, world)
        d = ctx.upload(a, bounds, rank)
    else:
        d = ctx.upload(a)
    # no grid call (the reference has none): the upload detects a 7- / 27-point
    # grid operator (each rank's z-slab of it) and gives it its stencil twin --
    # implicit columns, TMA-staged x planes, bitwise the CSR result
    if args.no_grid_hint:
        d.clear_grid()
    stencil = d.stencil_kind
    r0, r1 = d.row_begin, d.row_end
    b_loc = np.ascontiguousarray(b_full[r0 * m:r1 * m])
    B = ctx.multivector(d.n, m, b_loc)
    X = ctx.multivector(d.n, m)
    maxit = cfg["maxit"]

    def barrier():
        if dist is not None:
            dist.barrier()

    def step():
        X.fill(0.0)
        return P.solve(ctx, d, B, X, cfg["method"], cfg["formulation"], cfg["tol"], cfg["fixed"], maxit,
                       history=True)

    for _ in range(args.warmup):
        step()
    barrier()
    ctx.synchronize()
    launches0 = ctx.launches()
    reps = []
    with Clocks(local) as clk:
        for _ in range(args.steps):
            reps.append(step())
        ctx.synchronize()
    barrier()
    launches = ctx.launches() - launches0
    dev_ms = sum(r.loop_ms for r in reps)
    its = [r.iterations for r in reps]
    if dist is not None:
        import torch
        t = torch.tensor([dev_ms], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dev_ms = float(t.item())
    # strong scaling: the ranks together advance the whole n-row system's m RHS
    rhs_its = m * sum(its)
    value = rhs_its / (dev_ms / 1000.0)
    ms_per_step = dev_ms / args.steps
    clocks = clk.summary()
    peak, peak_src = peaks()

    # ---- byte model / achieved bandwidth over the whole iteration loop ----
    sched = P.method_schedule(cfg["method"], cfg["formulation"])
    v = sched["reads"] + sched["writes"]
    n_loc, nnz_loc = d.n, d.nnz
    b_iter = reps[0].compulsory_bytes / max(1, reps[0].iterations)   # this rank's bytes
    b_iter_eq3 = v * 8.0 * n_loc * m + sched["spmvs"] * P.spmv_traffic_bytes(n_loc, nnz_loc, m)
    hbm_gbs = b_iter * (sum(its) / args.steps) / (ms_per_step / 1000.0) / 1e9

    # ---- e2e through the host-buffer C ABI entry point ----
    e2e = None
    if not args.no_e2e:
        # host buffers in page-locked memory (DMA'd at link rate), as a
        # production caller of the C ABI would hold them
        bh = P.pinned_empty(n_loc * m)
        bh[:] = b_loc
        xh = P.pinned_empty(n_loc * m)
        xh[:] = 0.0
        e_its, e_time = [], 0.0
        P.solve_host(ctx, d, bh, xh, m, cfg["method"], cfg["formulation"], cfg["tol"], cfg["fixed"], maxit)
        barrier()
        for _ in range(args.steps):
            xh[:] = 0.0
            barrier()
            t0 = time.perf_counter()
            rep = P.solve_host(ctx, d, bh, xh, m, cfg["method"], cfg["formulation"], cfg["tol"], cfg["fixed"],
                               maxit)
            e_time += time.perf_counter() - t0
            e_its.append(rep.iterations)
        if dist is not None:
            import torch
            t = torch.tensor([e_time], dtype=torch.float64, device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            e_time = float(t.item())
        e2e = {"value": m * sum(e_its) / e_time, "unit": UNIT,
               "h2d_bytes_per_step": 2 * n_loc * m * 8,
               "d2h_bytes_per_step": n_loc * m * 8 + (max(e_its) + 1) * m * 8,
               "note": "mbg_solve_host: pinned host b/x0 uploaded, x + residual history downloaded, per solve "
                       "(bytes per rank)"}

    # ---- roofline of the dominant kernel (CUDA-event profile solve) ----
    # fixed mode over exactly the timed solve's iterations: every profiled
    # launch is a real one (no post-stop no-op launches in the averages)
    X.fill(0.0)
    prep, prof = P.solve_profile(ctx, d, B, X, cfg["method"], cfg["formulation"], cfg["tol"], True, its[0])
    total_ms = sum(v[1] for v in prof.values())
    dom = max(((k, v) for k, v in prof.items() if v[2] > 0), key=lambda kv: kv[1][1])
    dname, (dn, dms, dbytes) = dom
    achieved = dbytes / (dms / dn / 1000.0) / 1e9
    traffic = None
    ncu = ROOT / "profiles" / "ncu_dram_bytes.json"
    if ncu.exists():
        try:
            traffic = json.loads(ncu.read_text()).get(f"{cfg['name']}:{dname}")   # per launch, ncu --set full
        except Exception:
            traffic = None
    # gather-bound CSR SpMM (C5): its x gathers against the measured L2 gather
    # ceiling for their segment size (tools/l2_lab.cu -> profiles/l2_ceilings.json)
    gather = None
    ceil_f = ROOT / "profiles" / "l2_ceilings.json"
    if dname == "spmm" and not stencil and ceil_f.exists():
        try:
            ceil = json.loads(ceil_f.read_text())
            seg = max(16, 8 * m)
            cg = ceil["gather_GBps_by_segment_B"][str(min(256, seg))]
            if 8 * m < 16:   # 8-byte gathers move the same sectors as 16-byte ones
                cg *= 8.0 * m / 16.0
            gb = 8.0 * m * nnz_loc   # useful x bytes gathered per SpMM (one m-wide row of x per nonzero)
            ach = gb / (dms / dn / 1000.0) / 1e9
            gather = {"bound": "l2-gather", "achieved": ach, "peak": cg, "unit": "GB/s", "frac": ach / cg,
                      "bytes_per_launch": gb, "segment_B": 8 * m,
                      "peak_source": "tools/l2_lab.cu random L2-resident gathers of min(256, max(16, 8m))-byte "
                                     "segments (profiles/l2_ceilings.json)"}
        except Exception:
            gather = None
    kernels = {k: {"launches": v[0], "ms": round(v[1], 3), "share": round(v[1] / total_ms, 4),
                   "GB/s": round(v[2] / (v[1] / v[0] / 1000.0) / 1e9, 1) if v[2] > 0 else None}
               for k, v in prof.items()}

    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded counter RNG, DESIGN.md Inputs)",
        "config": config_dict(cfg, world, a.nnz()),
        "operator": (f"stencil twin ({stencil}-point slots, implicit columns)" if stencil else "CSR"),
        "iterations_per_step": its,
        "hbm": {"bytes_per_iteration_per_gpu": b_iter, "bytes_per_iteration_eq3_per_gpu": b_iter_eq3,
                "achieved_GBps_per_gpu": hbm_gbs, "peak_GBps": peak, "frac": hbm_gbs / peak,
                "rows_per_gpu": n_loc, "nnz_per_gpu": nnz_loc,
                "model": ("V*8*N*m + S*(16*N*m + 8*nnz + 4*N) (stencil twin: values + row masks, no columns)"
                          if stencil else "V*8*N*m + S*(16*N*m + 12*nnz + 4*N)") +
                         ", V = the formulation's transfers (Table 2 merged; fused: fewer)"},
        "clocks": clocks,
        "e2e": e2e,
        "gpu_launches": int(launches),
        "roofline": {"bound": "hbm", "kernel": dname, "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": traffic, "peak_source": peak_src,
                     "bytes_per_launch": dbytes, "avg_launch_ms": dms / dn, "launches": dn,
                     "profile_iterations": prep.iterations,
                     "how": "CUDA events around every launch of one fixed-mode profile solve over exactly the "
                            "timed solve's iterations, after the timed region"},
        "kernels": kernels,
    }
    if gather:
        line["roofline_l2_gather"] = gather
    if world == 1 and rank == 0 and not args.no_compare:
        line["variants"] = variants(P, ctx, a, cfg, d, B, X, peak, min(args.steps, 3))
        if cfg["name"] != "C2":
            del B, X
            line["c2_classical"] = c2_block(P, ctx, peak, min(args.steps, 3))
    if world == 1 and rank == 0 and not args.no_cpu_baseline:
        try:
            sys.path.insert(0, str(ROOT / "tests"))
            import oracle_ctypes as O
            a_o = O.Csr(a.n_rows, a.row_offsets, a.col_indices, a.values)   # bit-equal to the oracle's
            cb, _ = cpu_baseline(a_o, b_full, cfg, cpu_iters(cfg, args), steps=1)
            line["cpu_baseline"] = cb
        except Exception as e:  # noqa: BLE001
            line["cpu_baseline"] = {"value": None, "unit": UNIT, "error": str(e)[:200]}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
