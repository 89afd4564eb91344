"""The C++ API (include/mbstab_b200.hpp) compiled against the in-tree .so and
run on the GPU, as a reference C++ user would call it."""
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent


def build_demo(out: Path) -> None:
    lib = ROOT / "paper_1907_12874_b200"
    subprocess.run(["g++", "-std=c++20", "-O2", "-ffp-contract=off", f"-I{ROOT / 'include'}",
                    str(ROOT / "tests" / "cpp" / "api_smoke.cpp"), f"-L{lib}", "-lmbstab_b200",
                    f"-Wl,-rpath,{lib}", "-o", str(out)], check=True)


def test_cpp_api_compiles(tmp_path):
    build_demo(tmp_path / "api_smoke")


@pytest.mark.gpu
@pytest.mark.parametrize("auto_grid", ["1", "0"])
def test_cpp_api_runs(tmp_path, auto_grid):
    """auto_grid 1 = the product default: the upload detects the 7-point grid."""
    import os
    exe = tmp_path / "api_smoke"
    build_demo(exe)
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=300,
                       env={**os.environ, "MBG_AUTO_GRID": auto_grid})
    assert r.returncode == 0, r.stdout + r.stderr
    assert "cpp api ok" in r.stdout
