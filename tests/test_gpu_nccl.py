"""The NCCL transport on the one GPU this environment has: a 1-rank
communicator (ncclGetUniqueId -> ncclCommInitRank -> the solver's NCCL
barrier) around a partitioned upload with one part, in a child process so
NCCL's state does not leak into the other tests.  Multi-rank NCCL cannot run
here (NCCL rejects two ranks on one device); the multi-rank data path is
covered by the emulated communicator (test_gpu_multirank_local.py)."""
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu

HERE = Path(__file__).resolve().parent

SCRIPT = r"""
import sys
sys.path[:0] = [{root!r}, {tests!r}]
import numpy as np
import oracle_ctypes as O
import paper_1907_12874_b200 as P
ctx = P.Context(0)
ctx.init_comm(0, 1, P.comm_unique_id())
a = O.gen_stencil("convdiff7", 20, 18, 12, seed=1)
m = 8
b = O.rhs(a.n, m, 1)
d = ctx.upload(P.CsrMatrix(a.n, a.off, a.col, a.val), [0, a.n], 0)
d.set_grid(20, 18, 12)
B, X = ctx.multivector(a.n, m, b), ctx.multivector(a.n, m)
rep = P.solve(ctx, d, B, X, "pipebicgstab", "fused", 1e-8)
want = O.solve(a, b, m, "pipebicgstab", "fused", 1e-8)
assert rep.iterations == want["iterations"]
assert np.array_equal(rep.residual_history.view(np.int64), want["hist"].view(np.int64))
assert np.array_equal(X.download().view(np.int64), want["x"].view(np.int64))
print("nccl ok", rep.iterations)
"""


def test_nccl_single_rank_solve():
    code = SCRIPT.format(root=str(HERE.parent), tests=str(HERE))
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and "nccl ok" in r.stdout, r.stdout[-2000:] + r.stderr[-2000:]
