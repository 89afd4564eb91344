"""Out-of-bounds-write checking on the GPU (the stand-in for compute-sanitizer
memcheck, which this pool does not allow: profiles/r02h_compute_sanitizer_closed.txt).

The guard-zone build (csrc/Makefile `checked`, MBG_CHECKED) surrounds every
device allocation with 64 KB of 0xA5 bytes and verifies them on free and on
demand.  tools/sanitize_driver.py runs every hot kernel (CSR SpMM, both
stencil SpMMs, the group kernels of four methods, the one-launch small path,
the execute_group interpreter) on small inputs against the oracle under that
build; no guard may be touched.  A deliberate one-element overrun must be
caught (the mechanism works)."""
import os
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parent.parent
LIB = ROOT / "paper_1907_12874_b200" / "libmbstab_b200_checked.so"

CHECK = """
import sys
sys.path.insert(0, {root!r})
sys.path.insert(0, {tools!r})
import runpy
runpy.run_path({driver!r}, run_name="__main__")
import paper_1907_12874_b200 as P
v = P.debug_guard_check()
print("violations", v)
assert v == 0, v
c = P.Context(0)
X = c.multivector(1000, 4)
P.debug_write_past_end(X)
v = P.debug_guard_check()
print("after overrun", v)
assert v == 1, v
print("checked ok")
"""


@pytest.fixture(scope="module")
def checked_lib():
    if not LIB.exists():
        r = subprocess.run(["make", "-s", "-j", str(os.cpu_count() or 4), "-C",
                            str(ROOT / "paper_1907_12874_b200" / "csrc"), "checked"],
                           capture_output=True, text=True, timeout=1500)
        assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
    return LIB


@pytest.mark.parametrize("z", ["0", "3"])
def test_no_out_of_bounds_writes(checked_lib, z):
    code = CHECK.format(root=str(ROOT), tools=str(ROOT / "tools"), driver=str(ROOT / "tools" / "sanitize_driver.py"))
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=900,
                       env={**os.environ, "MBG_CHECKED": "1", "MBG_STENCIL_Z": z})
    assert r.returncode == 0 and "checked ok" in r.stdout, r.stdout[-3000:] + r.stderr[-3000:]
