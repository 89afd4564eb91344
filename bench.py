#!/usr/bin/env python
"""Benchmark: RHS-iterations/s of the multi-RHS BiCGStab hot path on B200.

Default workload = BASELINE.json configs[1] (config C2): classical merged
BiCGStab, nonsymmetric 7-point convection-diffusion on a 128^3 grid, m=8 RHS
(seed 1), rel tol 1e-8, max 1000 iterations.  One step = one full solve from
x0 = 0 to convergence.  With N GPUs (torchrun) the grid is extended in z to
128x128x(128N) and split in z-slabs, one 128^3 slab per GPU (weak scaling).

  value   RHS-iterations/s over the timed steps (device CUDA events, inputs
          resident in HBM, max over ranks)
  e2e     same metric through the C ABI with HOST buffers: b and x0 uploaded,
          x and the history downloaded inside the timed region
  roofline dominant kernel of the iteration loop (CUDA-event profile solve)
  cpu_baseline  the reference's own kernels (oracle/_ref) on the host cores

`--impl reference` times the reference CPU implementation (oracle/_ref: the
reference's core::spmv + kernels::execute_group driving the restated merged
solver) on the same config; rank 0 only.
"""
from __future__ import annotations

import argparse
import json
import os
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


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=5)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--method", default="bicgstab", choices=["bicgstab", "rbicgstab", "pipebicgstab"])
    p.add_argument("--formulation", default="fused", choices=["merged", "basic", "fused"],
                   help="fused (default): the Alg. 2 merged listing with theta=(s,s) computed in the pass "
                        "that produces s -- same 18 transfers and reduction layout, bitwise-identical results")
    p.add_argument("--no-compare", action="store_true", help="skip the paper-listing merged comparison run")
    p.add_argument("--grid", type=int, default=128, help="per-GPU grid edge (config C2: 128)")
    p.add_argument("--m", type=int, default=8)
    p.add_argument("--tol", type=float, default=1e-8)
    p.add_argument("--maxit", type=int, default=1000)
    p.add_argument("--fixed", type=int, default=0, help="fixed iteration count instead of tol")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--cpu-iters", type=int, default=10)
    p.add_argument("--no-grid-hint", action="store_true", help="plain CSR SpMM (no stencil twin)")
    return p.parse_args()


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def workload_desc(args, world):
    g = args.grid
    mode = f"fixed {args.fixed} iterations" if args.fixed else f"rel tol {args.tol:g}, max {args.maxit}"
    return (f"C2: {args.method} {args.formulation}, conv-diff 7-pt {g}x{g}x{g * world} "
            f"(z-slab per GPU), m={args.m} RHS u[-1,1] seed 1, x0=0, {mode}")


def build_problem(args, world):
    import paper_1907_12874_b200 as P
    g = args.grid
    a = P.gen_stencil("convdiff7", g, g, g * world, seed=1)
    b = P.gen_rhs(a.n_rows, args.m, 1)
    return a, b


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


def cpu_baseline(a_np, b, args, steps=1):
    """Reference kernels (oracle/_ref) on the host cores, bounded sample."""
    sys.path.insert(0, str(ROOT / "tests"))
    import oracle_ctypes as O
    a = O.Csr(a_np.n_rows, a_np.row_offsets, a_np.col_indices, a_np.values)
    threads = os.cpu_count() or 1
    iters = args.cpu_iters
    if O.ref_available():
        vals = []
        for _ in range(steps):
            _, its, secs = O.ref_solve(a, b, args.m, args.method, tol=args.tol, fixed=True, maxit=iters,
                                       threads=threads, timing=True)
            vals.append(args.m * its / secs)
        kind = "reference"
        sample = (f"same matrix and RHS, {iters} fixed iterations of the restated merged {args.method} on the "
                  f"reference's core::spmv + kernels::execute_group (oracle/_ref), threads={threads}, "
                  f"setup excluded")
    else:
        vals = []
        for _ in range(steps):
            t = time.perf_counter()
            O.solve(a, b, args.m, args.method, args.formulation, args.tol, True, iters)
            vals.append(args.m * iters / (time.perf_counter() - t))
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


def run_reference(args):
    world, rank, _ = dist_env()
    if rank != 0:
        return
    a, b = build_problem(args, 1)
    steps = []
    for i in range(args.warmup + args.steps):
        cb, vals = cpu_baseline(a, b, args, steps=1)
        if i >= args.warmup:
            steps.append(vals[0])
    value = float(np.mean(steps))
    cb["value"] = value
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1000.0 * args.m * args.cpu_iters / value,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded counter RNG, DESIGN.md Inputs)",
        "config": {"workload": workload_desc(args, args.gpus),
                   "step": f"{args.cpu_iters} fixed iterations on one 128^3 slab (bounded sample; the CPU's "
                           "slab-RHS-iterations/s do not depend on how many slabs the job has)"},
        "cpu_baseline": cb,
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
        return
    import paper_1907_12874_b200 as P
    world, rank, local = dist_env()
    dist = None
    if world > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    a, b_full = build_problem(args, world)
    m = args.m
    ctx = P.Context(local)
    if world > 1:
        nid = [P.comm_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(nid, src=0)
        ctx.init_comm(rank, world, nid[0])
        slab = args.grid ** 3
        bounds = [p * slab for p in range(world + 1)]
        d = ctx.upload(a, bounds, rank)
    else:
        d = ctx.upload(a)
    # structured-grid hint (mbg_csr_set_grid, global grid): the 7-point operator
    # (each rank's z-slab of it) gets its stencil twin -- implicit columns,
    # TMA-staged x planes, bitwise the CSR result
    if not args.no_grid_hint:
        d.set_grid(args.grid, args.grid, args.grid * world)
    stencil = d.stencil_kind
    r0, r1 = d.row_begin, d.row_end
    b_loc = np.ascontiguousarray(b_full[r0 * m:r1 * m])
    B = ctx.multivector(d.n, m, b_loc)
    X = ctx.multivector(d.n, m)
    fixed = bool(args.fixed)
    maxit = args.fixed if fixed else args.maxit

    def barrier():
        if dist is not None:
            dist.barrier()

    def step():
        X.fill(0.0)
        return P.solve(ctx, d, B, X, args.method, args.formulation, args.tol, fixed, maxit, history=True)

    for _ in range(args.warmup):
        step()
    barrier()
    ctx.synchronize()
    launches0 = ctx.launches()
    reps = []
    with Clocks(local) as clk:
        t_wall = time.perf_counter()
        for _ in range(args.steps):
            reps.append(step())
        ctx.synchronize()
        t_wall = time.perf_counter() - t_wall
    barrier()
    launches = ctx.launches() - launches0
    dev_ms = sum(r.loop_ms for r in reps)
    # the paper's merged listing verbatim, same workload (reported beside)
    compare = None
    if not args.no_compare and args.formulation != "merged":
        creps = []
        for i in range(args.warmup + args.steps):
            X.fill(0.0)
            rr = P.solve(ctx, d, B, X, args.method, "merged", args.tol, fixed, maxit, history=False)
            if i >= args.warmup:
                creps.append(rr)
        cms = sum(r.loop_ms for r in creps)
        compare = {"formulation": "merged (paper listing)",
                   "value": world * m * sum(r.iterations for r in creps) / (cms / 1000.0),
                   "ms_per_step": cms / len(creps)}
    its = [r.iterations for r in reps]
    if dist is not None:
        import torch
        t = torch.tensor([dev_ms], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dev_ms = float(t.item())
    # weak scaling: every rank advances its own 128^3-row slab of the m RHS per
    # iteration, so the job processes world * m slab-RHS-iterations per iteration
    rhs_its = world * m * sum(its)
    value = rhs_its / (dev_ms / 1000.0)
    ms_per_step = dev_ms / args.steps
    clocks = clk.summary()

    # ---- byte model / achieved bandwidth over the whole iteration loop ----
    sched = P.method_schedule(args.method, args.formulation)
    v = sched["reads"] + sched["writes"]
    n_loc, nnz_loc = d.n, d.nnz
    # the solver's own byte model: formulation transfers + SpMMs, 12 B/nnz for
    # CSR, 8 B/nnz + 4 B/row mask for the stencil twin (no column indices)
    b_iter = reps[0].compulsory_bytes / max(1, reps[0].iterations)
    b_iter_eq3 = v * 8.0 * n_loc * m + sched["spmvs"] * P.spmv_traffic_bytes(n_loc, nnz_loc, m)
    hbm_gbs = b_iter * (sum(its) / args.steps) / (ms_per_step / 1000.0) / 1e9
    peak, peak_src = peaks()

    # ---- e2e through the host-buffer C ABI entry point ----
    e2e = None
    if not args.no_e2e:
        # host buffers in page-locked memory (DMA'd at link rate), as a
        # production caller of the C ABI would hold them
        bh = P.pinned_empty(n_loc * m)
        bh[:] = b_loc
        b_loc = bh
        xh = P.pinned_empty(n_loc * m)
        xh[:] = 0.0
        e_its, e_time = [], 0.0
        P.solve_host(ctx, d, b_loc, xh, m, args.method, args.formulation, args.tol, fixed, maxit)
        barrier()
        for _ in range(args.steps):
            xh[:] = 0.0
            t0 = time.perf_counter()
            rep = P.solve_host(ctx, d, b_loc, xh, m, args.method, args.formulation, args.tol, fixed, maxit)
            e_time += time.perf_counter() - t0
            e_its.append(rep.iterations)
        if dist is not None:
            import torch
            t = torch.tensor([e_time], dtype=torch.float64, device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            e_time = float(t.item())
        e2e = {"value": world * m * sum(e_its) / e_time, "unit": UNIT,
               "h2d_bytes_per_step": 2 * n_loc * m * 8,
               "d2h_bytes_per_step": n_loc * m * 8 + (max(e_its) + 1) * m * 8,
               "note": "mbg_solve_host: pinned host b/x0 uploaded, x + residual history downloaded, per solve"}

    # ---- roofline of the dominant kernel (CUDA-event profile solve) ----
    X.fill(0.0)
    prep, prof = P.solve_profile(ctx, d, B, X, args.method, args.formulation, args.tol, fixed, maxit)
    total_ms = sum(v[1] for v in prof.values())
    dom = max(((k, v) for k, v in prof.items() if v[2] > 0), key=lambda kv: kv[1][1])
    dname, (dn, dms, dbytes) = dom
    achieved = dbytes / (dms / dn / 1000.0) / 1e9
    traffic = None
    ncu = ROOT / "profiles" / "ncu_dram_bytes.json"
    if ncu.exists():
        try:
            traffic = json.loads(ncu.read_text()).get(dname)
        except Exception:
            traffic = None
    kernels = {k: {"launches": v[0], "ms": round(v[1], 3), "share": round(v[1] / total_ms, 4),
                   "GB/s": round(v[2] / (v[1] / v[0] / 1000.0) / 1e9, 1) if v[2] > 0 else None}
               for k, v in prof.items()}

    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded counter RNG, DESIGN.md Inputs)",
        "config": {"workload": workload_desc(args, world), "rows": int(a.n_rows), "nnz": int(a.nnz()),
                   "m": m, "method": args.method, "formulation": args.formulation,
                   "parallelism": f"row-partition z-slabs x{world}",
                   "operator": (f"stencil twin ({stencil}-point slots, implicit columns)" if stencil
                                else "CSR"),
                   "units": "RHS-iterations of one 128^3-row slab, summed over GPUs (weak scaling)",
                   "l2": f"inputs larger than L2 (working set {((8 + 2) * n_loc * m * 8 + 12 * nnz_loc) / 1e9:.2f} GB/GPU)"},
        "iterations_per_step": its,
        "merged_listing": compare,
        "hbm": {"bytes_per_iteration": b_iter, "bytes_per_iteration_eq3": b_iter_eq3,
                "achieved_GBps": hbm_gbs, "peak_GBps": peak, "frac": hbm_gbs / peak,
                "model": ("V*8*N*m + 2*(16*N*m + 8*nnz + 4*N) (stencil twin: values + row masks, no columns)"
                          if stencil else "V*8*N*m + 2*(16*N*m + 12*nnz + 4*N)") +
                         ", V = the formulation's transfers (Table 2 merged; fused: fewer)"},
        "clocks": clocks,
        "e2e": e2e,
        "gpu_launches": int(launches),
        "roofline": {"bound": "hbm", "kernel": dname, "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": traffic, "peak_source": peak_src,
                     "bytes_per_launch": dbytes, "avg_launch_ms": dms / dn,
                     "how": "CUDA events around every launch of one profile solve after the timed region"},
        "kernels": kernels,
    }
    if world == 1 and rank == 0 and not args.no_cpu_baseline:
        try:
            cb, _ = cpu_baseline(a, b_full, args, steps=1)
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
