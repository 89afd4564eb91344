"""Multi-rank host logic on CPU (gloo, world_size 2 and 3): each rank builds the
product's halo plan for its row block, exchanges halo rows with the plan's
send lists / receive windows, multiplies its local renumbered CSR (oracle
arithmetic) and sums its exact-dot limbs with an int64 allreduce -- the data
path the NCCL ranks run on GPUs.  Results must equal the single-process
oracle bit for bit."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, case, q):
    import sys
    from pathlib import Path
    root = Path(__file__).resolve().parent.parent
    sys.path[:0] = [str(root), str(root / "tests")]
    import oracle_ctypes as O
    import paper_1907_12874_b200 as P

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    try:
        m = 3
        if case == "banded":
            a = P.gen_banded(20_000, 3000, 8, 20, 4)
            n = a.n_rows
            bounds = [n * p // world for p in range(world + 1)]
        else:  # z-slab partition of a 27-point stencil
            nx, ny, nz = 9, 8, 6 * world
            a = P.gen_stencil("stencil27", nx, ny, nz, seed=2)
            n = a.n_rows
            bounds = [p * nx * ny * 6 for p in range(world + 1)]
        x = np.random.default_rng(42).standard_normal(n * m)   # every rank can regenerate x ...
        r0, r1 = bounds[rank], bounds[rank + 1]

        def exchange_and_multiply(pl):
            # ... but only uses its own rows plus what the halo exchange delivers
            xl = np.zeros((pl["n_own"] + pl["n_halo"]) * m)
            xl[: pl["n_own"] * m] = x[r0 * m:r1 * m]
            reqs, bufs = [], []
            for peer in pl["peers"]:
                if len(peer["send_rows"]):
                    rows = peer["send_rows"].astype(np.int64)
                    buf = torch.from_numpy(xl.reshape(-1, m)[rows].copy())
                    bufs.append(buf)
                    reqs.append(dist.isend(buf, dst=peer["part"]))
            recv = []
            for peer in pl["peers"]:
                if peer["recv_count"]:
                    buf = torch.zeros(peer["recv_count"], m, dtype=torch.float64)
                    recv.append((peer, buf))
                    reqs.append(dist.irecv(buf, src=peer["part"]))
            for r in reqs:
                r.wait()
            for peer, buf in recv:
                o = (pl["n_own"] + peer["recv_offset"]) * m
                xl[o:o + buf.numel()] = buf.numpy().reshape(-1)
            return O.spmv(O.Csr(pl["n_own"], pl["off"].astype(np.int64), pl["col"], pl["val"]), xl, m)

        pl = P.halo_plan(a, bounds, rank)
        glob = O.Csr(n, a.row_offsets, a.col_indices, a.values)
        y_ref = O.spmv(glob, x, m)[r0 * m:r1 * m]
        spmv_ok = bool(np.array_equal(exchange_and_multiply(pl).view(np.int64), y_ref.view(np.int64)))
        # A^T x with the transpose plan (IBiCGStab's f0) == spmv_transpose, bitwise
        yt_ref = O.spmv_transpose(glob, x, m)[r0 * m:r1 * m]
        plt = P.halo_plan(a, bounds, rank, transpose=True)
        spmvt_ok = bool(np.array_equal(exchange_and_multiply(plt).view(np.int64), yt_ref.view(np.int64)))

        # exact dot over the partition: int64 limb allreduce
        b = np.random.default_rng(7).standard_normal(n * m) * np.exp2(
            np.random.default_rng(8).integers(-80, 80, n * m))
        limbs = P.exact_accumulate(x[r0 * m:r1 * m], b[r0 * m:r1 * m], m)
        t = torch.from_numpy(limbs)
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
        got = P.exact_round(t.numpy(), m)
        want = O.dot_exact(x, b, m)
        dot_ok = bool(np.array_equal(got.view(np.int64), want.view(np.int64)))
        q.put((rank, spmv_ok, dot_ok, len(pl["peers"]), spmvt_ok))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("case", ["banded", "zslab27"])
def test_partitioned_spmv_and_exact_allreduce(world, case):
    ctx = mp.get_context("spawn")
    q = ctx.SimpleQueue()
    port = _free_port()
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    procs = [ctx.Process(target=_worker, args=(r, world, port, case, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=300)
        assert p.exitcode == 0
    res = sorted(q.get() for _ in range(world))
    assert all(r[1] for r in res), f"partitioned spmv mismatch: {res}"
    assert all(r[2] for r in res), f"limb allreduce mismatch: {res}"
    assert all(r[3] >= 1 for r in res)
    assert all(r[4] for r in res), f"partitioned A^T x mismatch: {res}"
