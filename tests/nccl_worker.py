"""Worker for tests/test_gpu_nccl_multi.py: one process per GPU under
torch.distributed.run.  Every rank joins a real NCCL communicator through
mbg_ctx_init_comm, solves its z-slab (or row block) of the system with the
captured-graph solver (ncclSend/Recv halo + ncclAllReduce of int64 limbs),
and rank 0 compares the gathered solution and the history with a 1-GPU solve
and with the CPU oracle, bit for bit.  Test infrastructure (imports oracle/)."""
import os
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import oracle_ctypes as O  # noqa: E402
import paper_1907_12874_b200 as P  # noqa: E402

CASES = [
    # (kind, dims, m, method, formulation, fixed iterations (0 = tol 1e-8))
    ("stencil27", (48, 40, 32), 16, "rbicgstab", "fused", 0),      # C3-shaped z-slabs, stencil twin
    ("convdiff7", (64, 48, 40), 32, "pipebicgstab", "fused", 30),  # C4-shaped: overlapped allreduce
    ("convdiff7", (64, 48, 40), 8, "bicgstab", "fused", 0),        # C2-shaped classical
    ("banded", 200_000, 8, "bicgstab", "merged", 25),              # C5-shaped row blocks, CSR halo
]


def main():
    rank, world, local = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"]), int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    ctx = P.Context(local)
    nid = [P.comm_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(nid, src=0)
    ctx.init_comm(rank, world, nid[0])
    single = P.Context(local) if rank == 0 else None
    fails = []
    for kind, dims, m, method, form, fixed in CASES:
        if kind == "banded":
            a = O.gen_banded(dims, 4096, 16, 32, 4)
            bounds = [a.n * p // world for p in range(world + 1)]
        else:
            a = O.gen_stencil(kind, *dims, seed=2)
            nx, ny, nz = dims
            bounds = [(nz * p // world) * nx * ny for p in range(world + 1)]
        b = O.rhs(a.n, m, 3)
        pa = P.CsrMatrix(a.n, a.off, a.col, a.val)
        d = ctx.upload(pa, bounds, rank)
        if kind != "banded":
            d.set_grid(*dims)
        r0, r1 = d.row_begin, d.row_end
        B = ctx.multivector(d.n, m, b[r0 * m:r1 * m])
        X = ctx.multivector(d.n, m)
        maxit = fixed or 1000
        rep = P.solve(ctx, d, B, X, method, form, 1e-8, bool(fixed), maxit)
        parts = [None] * world
        dist.all_gather_object(parts, X.download())
        if rank == 0:
            x = np.concatenate(parts)
            d1 = single.upload(pa)
            if kind != "banded":
                d1.set_grid(*dims)
            B1, X1 = single.multivector(a.n, m, b), single.multivector(a.n, m)
            rep1 = P.solve(single, d1, B1, X1, method, form, 1e-8, bool(fixed), maxit)
            want = O.solve(a, b, m, method, form, 1e-8, bool(fixed), maxit)
            tag = f"{kind}{dims} m={m} {method} {form} world={world}"
            ok = (rep.iterations == rep1.iterations == want["iterations"] and
                  np.array_equal(rep.residual_history.view(np.int64), rep1.residual_history.view(np.int64)) and
                  np.array_equal(rep.residual_history.view(np.int64), want["hist"].view(np.int64)) and
                  np.array_equal(x.view(np.int64), X1.download().view(np.int64)) and
                  np.array_equal(x.view(np.int64), want["x"].view(np.int64)))
            print(f"{'ok  ' if ok else 'FAIL'} {tag}: iterations {rep.iterations}/{rep1.iterations}/"
                  f"{want['iterations']}", flush=True)
            if not ok:
                fails.append(tag)
        dist.barrier()
    if rank == 0:
        print("ALL OK" if not fails else f"FAILED: {fails}", flush=True)
    dist.barrier()
    ctx.close()
    dist.destroy_process_group()
    sys.exit(1 if fails else 0)


if __name__ == "__main__":
    main()
