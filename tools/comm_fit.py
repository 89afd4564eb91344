#!/usr/bin/env python
"""Fit the communication terms of the paper's time model on this box
(PAPER.md:596-613 T_L, 650-669 T_G and gamma, 690-706 Eq. 13).

Run one process per GPU:
    python -m torch.distributed.run --nproc-per-node N --master-addr 127.0.0.1 \
        tools/comm_fit.py --out gpurun_out/comm_fit_pN.json

  T_G(p, l)  ncclAllReduce (int64 sum) of l limb words -- the solver's
             reduction-point message (k dots x m columns x 72 words)
  T_L(l)     halo exchange of l bytes with both z neighbours (ncclSend/Recv
             pairs, the z-slab pattern of the stencil SpMM)
  gamma      overlap factor (T_calc^async + T_comm^async - T_calc^sync) / T_comm^sync
             for the product's SpMM (C3-shaped slab, stencil twin) running on
             its stream while the halo / allreduce runs on another
All times: CUDA events / synchronised host clocks, median of --reps, MAX over
ranks.  At N = 1 the collectives are local copies (recorded, not fitted).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402


def timed(fn, reps, stream=None):
    ts = []
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    for _ in range(reps):
        dist.barrier()
        torch.cuda.synchronize()
        t = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t)
    v = torch.tensor([statistics.median(ts)], dtype=torch.float64, device="cuda")
    dist.all_reduce(v, op=dist.ReduceOp.MAX)
    return float(v.item())


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=str(ROOT / "gpurun_out" / "comm_fit.json"))
    ap.add_argument("--reps", type=int, default=20)
    args = ap.parse_args()
    rank, world, local = int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), \
        int(os.environ.get("LOCAL_RANK", 0))
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", "29533")
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local), rank=rank, world_size=world)
    rec = {"world": world, "T_G": {}, "T_L": {}, "gamma": {}}

    # T_G: limb allreduce of k dots x m columns x 72 int64 words
    for m in (1, 8, 16, 32):
        for k in (1, 3, 4):
            words = k * m * 72
            buf = torch.ones(words, dtype=torch.int64, device="cuda")
            rec["T_G"][f"m{m}_k{k}_{words * 8}B"] = timed(lambda: dist.all_reduce(buf), args.reps)

    # T_L: z-neighbour halo exchange of one plane per side
    def halo(nbytes):
        n = nbytes // 8
        send = [torch.ones(n, dtype=torch.float64, device="cuda") for _ in range(2)]
        recv = [torch.empty(n, dtype=torch.float64, device="cuda") for _ in range(2)]

        def run():
            ops = []
            if rank > 0:
                ops += [dist.P2POp(dist.isend, send[0], rank - 1), dist.P2POp(dist.irecv, recv[0], rank - 1)]
            if rank < world - 1:
                ops += [dist.P2POp(dist.isend, send[1], rank + 1), dist.P2POp(dist.irecv, recv[1], rank + 1)]
            if ops:
                for r in dist.batch_isend_irecv(ops):
                    r.wait()
        return run

    planes = {"C3_plane_192x192_m16": 192 * 192 * 16 * 8, "C4_plane_320x320_m32": 320 * 320 * 32 * 8,
              "C2_plane_128x128_m8": 128 * 128 * 8 * 8}
    for name, nb in planes.items():
        rec["T_L"][f"{name}_{nb}B"] = timed(halo(nb), args.reps) if world > 1 else None

    # gamma: the product's SpMM (one rank's C3 slab on the stencil twin) with
    # the halo exchange / the limb allreduce on another stream
    import paper_1907_12874_b200 as P
    nz = max(1, 192 // world)
    a = P.gen_stencil("stencil27", 192, 192, nz, seed=2)
    ctx = P.Context(local)
    d = ctx.upload(a)
    d.set_grid(192, 192, nz)
    X = ctx.multivector(a.n_rows, 16, P.gen_rhs(a.n_rows, 16, 2))
    Y = ctx.multivector(a.n_rows, 16)
    calc = lambda: (P.spmv(ctx, d, X, Y), ctx.synchronize())  # noqa: E731
    t_calc = timed(calc, args.reps)
    side = torch.cuda.Stream()
    for cname, comm in (("halo_C3_plane", halo(planes["C3_plane_192x192_m16"]) if world > 1 else None),
                        ("allreduce_m16_k4", None)):
        if cname.startswith("allreduce"):
            buf = torch.ones(4 * 16 * 72, dtype=torch.int64, device="cuda")
            comm = lambda: dist.all_reduce(buf)  # noqa: E731
        if comm is None:
            continue
        t_comm = timed(comm, args.reps)

        def both():
            with torch.cuda.stream(side):
                comm()
            P.spmv(ctx, d, X, Y)
            ctx.synchronize()
            side.synchronize()
        t_both = timed(both, args.reps)
        rec["gamma"][cname] = {"T_calc_sync_s": t_calc, "T_comm_sync_s": t_comm, "T_async_s": t_both,
                               "gamma": (t_both - t_calc) / t_comm if t_comm > 0 else None}
    if rank == 0:
        Path(args.out).parent.mkdir(parents=True, exist_ok=True)
        Path(args.out).write_text(json.dumps(rec, indent=1))
        print(json.dumps(rec))
    ctx.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
