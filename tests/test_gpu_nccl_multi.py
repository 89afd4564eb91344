"""Real multi-rank NCCL (skipped unless the box has >= 2 GPUs): the captured
solver graph replays ncclSend/ncclRecv halo exchanges and ncclAllReduce of
int64 limbs across processes, one per GPU, and the history and the gathered
solution must equal the 1-GPU solve and the oracle bit for bit (C3-shaped
z-slabs on the stencil twin, C4-shaped Pipelined with the overlapped
allreduce, C2-shaped classical, C5-shaped CSR row blocks)."""
import os
import socket
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
HERE = Path(__file__).resolve().parent


def _worlds():
    import torch
    n = torch.cuda.device_count()
    return sorted({w for w in (2, n) if 2 <= w <= min(n, 8)})


@pytest.mark.parametrize("world", [2, 0])
def test_nccl_multi_rank_bitwise(world):
    worlds = _worlds()
    if not worlds:
        pytest.skip("needs >= 2 GPUs (this box has fewer)")
    if world == 0:
        world = max(worlds)
        if world == 2:
            pytest.skip("all-GPU case equals the 2-GPU case here")
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), str(HERE / "nccl_worker.py")]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=1500, cwd=str(HERE.parent),
                       env={**os.environ, "NCCL_DEBUG": "WARN"})
    assert r.returncode == 0 and "ALL OK" in r.stdout, r.stdout[-3000:] + r.stderr[-3000:]
