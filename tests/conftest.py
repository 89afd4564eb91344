import os
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(Path(__file__).resolve().parent))


# The upload detects 7- / 27-point grid operators and gives them the stencil
# twin (tests/test_gpu_autogrid.py covers that).  Everywhere else the tests
# decide themselves which SpMM a matrix takes (set_grid = stencil twin, none =
# the CSR kernels), so the detection is off unless a test turns it on.
os.environ.setdefault("MBG_AUTO_GRID", "0")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")
    config.addinivalue_line("markers", "slow: large-size cases")
    # test infrastructure only: compile the sm_100a library (nvcc cross-compiles
    # without a GPU) if a fresh checkout runs the tests before __graft_entry__.build();
    # the product itself never builds or falls back at run time
    lib = ROOT / "paper_1907_12874_b200" / "libmbstab_b200.so"
    if not lib.exists():
        import shutil
        import subprocess
        if shutil.which("make") and (shutil.which("nvcc") or Path("/usr/local/cuda/bin/nvcc").exists()):
            subprocess.run(["make", "-s", "-j", str(os.cpu_count() or 4), "-C",
                            str(ROOT / "paper_1907_12874_b200" / "csrc")], check=False)


@pytest.fixture(scope="session")
def ctx():
    import paper_1907_12874_b200 as P
    c = P.Context(0)
    yield c
    c.close()
