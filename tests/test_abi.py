"""The C-ABI library loads without a GPU and exports every symbol declared in
include/*.h; device entry points fail cleanly (no crash) where there is none."""
import ctypes as C
import re
from pathlib import Path

import pytest
import torch  # noqa: F401  -- load torch before this file dlopens the C-ABI library repeatedly

import paper_1907_12874_b200 as P

ROOT = Path(__file__).resolve().parent.parent


def declared_symbols():
    syms = set()
    for h in (ROOT / "include").glob("*.h"):
        text = re.sub(r"/\*.*?\*/", "", h.read_text(), flags=re.S)
        syms |= set(re.findall(r"\b(mbg_[a-z0-9_]+)\s*\(", text))
    return sorted(syms)


def test_header_declares_the_api():
    syms = declared_symbols()
    for s in ["mbg_spmv", "mbg_execute_group", "mbg_solve", "mbg_solve_host", "mbg_csr_upload",
              "mbg_analyze_traffic", "mbg_ctx_init_comm"]:
        assert s in syms


@pytest.mark.parametrize("sym", declared_symbols())
def test_symbol_exported(sym):
    lib = C.CDLL(str(P._lib.LIB_PATH))
    assert hasattr(lib, sym), f"{sym} declared in include/ but not exported"


def test_library_is_sm100a():
    import subprocess
    out = subprocess.run(["cuobjdump", "--list-elf", str(P._lib.LIB_PATH)], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_version_and_errors_without_gpu():
    import torch
    assert P.lib().mbg_version().decode().startswith("mbstab_b200")
    if not torch.cuda.is_available():
        with pytest.raises((RuntimeError, ValueError)):
            P.Context(0)
