"""ctypes bindings for the CPU oracle (oracle/liborc.so) and the reference
kernels compiled from their own sources (oracle/_ref/libmbstab_ref.so).

Test infrastructure: imported only by tests/, __graft_entry__.smoke() and
bench.py's CPU legs -- never by the product package.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
ORACLE_SO = ROOT / "oracle" / "liborc.so"
REF_SO = ROOT / "oracle" / "_ref" / "libmbstab_ref.so"

_i64p = np.ctypeslib.ndpointer(np.int64, flags="C_CONTIGUOUS")
_i32p = np.ctypeslib.ndpointer(np.int32, flags="C_CONTIGUOUS")
_f64p = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")


class OrcCsr(C.Structure):
    _fields_ = [("n", C.c_int64), ("nnz", C.c_int64), ("off", C.POINTER(C.c_int64)),
                ("col", C.POINTER(C.c_int32)), ("val", C.POINTER(C.c_double))]


class OrcReport(C.Structure):
    _fields_ = [("iterations", C.c_int), ("converged", C.c_int), ("breakdown", C.c_int),
                ("breakdown_iter", C.c_int), ("breakdown_col", C.c_int)]


METHODS = {"bicgstab": 0, "rbicgstab": 1, "pipebicgstab": 2, "ibicgstab": 3, "pbicgstab": 4, "ppipebicgstab": 5}
FORMULATIONS = {"merged": 0, "basic": 1, "fused": 0}  # fused rounds exactly like merged


def build_oracle() -> None:
    """Compile oracle/ (and oracle/_ref when /root/reference is present)."""
    import subprocess
    subprocess.run(["make", "-s", "-C", str(ROOT / "oracle")], check=True)


_orc = None
_ref = None


def orc() -> C.CDLL:
    global _orc
    if _orc is None:
        if not ORACLE_SO.exists():
            build_oracle()
        lib = C.CDLL(str(ORACLE_SO))
        lib.orc_hash4.restype = C.c_uint64
        lib.orc_hash4.argtypes = [C.c_uint64] * 4
        lib.orc_u11.restype = C.c_double
        lib.orc_u11.argtypes = [C.c_uint64] * 4
        lib.orc_gen_stencil.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, C.c_uint64, C.POINTER(OrcCsr)]
        lib.orc_gen_banded.argtypes = [C.c_int64, C.c_int64, C.c_int, C.c_int, C.c_uint64, C.POINTER(OrcCsr)]
        lib.orc_csr_free.argtypes = [C.POINTER(OrcCsr)]
        lib.orc_rhs.argtypes = [C.c_int64, C.c_int, C.c_uint64, _f64p]
        lib.orc_spmv.argtypes = [C.POINTER(OrcCsr), C.c_int, _f64p, _f64p]
        lib.orc_dot_exact.argtypes = [C.c_int64, C.c_int, _f64p, _f64p, _f64p]
        lib.orc_sum_exact.restype = C.c_double
        lib.orc_sum_exact.argtypes = [C.c_int64, _f64p]
        lib.orc_update.argtypes = [C.c_int64, C.c_int, C.c_int, C.POINTER(C.c_void_p),
                                   C.POINTER(C.c_void_p), _f64p]
        lib.orc_solve.argtypes = [C.POINTER(OrcCsr), C.c_int, _f64p, _f64p, C.c_int, C.c_int,
                                  C.c_double, C.c_int, C.c_int, _f64p, C.POINTER(OrcReport)]
        lib.orc_solve_pc.argtypes = [C.POINTER(OrcCsr), C.c_int, _f64p, _f64p, C.c_int, C.c_int, C.c_int,
                                     C.c_double, C.c_int, C.c_int, _f64p, C.POINTER(OrcReport)]
        lib.orc_method_preconditioned.argtypes = [C.c_int]
        lib.orc_spmv_transpose.argtypes = [C.POINTER(OrcCsr), C.c_int, _f64p, _f64p]
        lib.orc_num_threads.restype = C.c_int
        _orc = lib
    return _orc


def ref_available() -> bool:
    return REF_SO.exists()


def ref() -> C.CDLL:
    global _ref
    if _ref is None:
        lib = C.CDLL(str(REF_SO))
        lib.ref_last_error.restype = C.c_char_p
        lib.ref_gen_poisson_7pt.argtypes = [C.c_int, C.c_int, C.c_int, C.POINTER(C.c_int64),
                                            C.c_void_p, C.c_void_p, C.c_void_p]
        lib.ref_validate.argtypes = [C.c_int64, _i64p, _i32p, _f64p]
        lib.ref_gen_poisson_5pt.argtypes = [C.c_int, C.c_int, C.POINTER(C.c_int64), C.c_void_p, C.c_void_p,
                                            C.c_void_p]
        lib.ref_spmv.argtypes = [C.c_int64, _i64p, _i32p, _f64p, C.c_int, _f64p, _f64p, C.c_int]
        lib.ref_spmv_transpose.argtypes = [C.c_int64, _i64p, _i32p, _f64p, C.c_int, _f64p, _f64p]
        lib.ref_read_matrix_market.argtypes = [C.c_char_p, C.POINTER(C.c_int64), C.POINTER(C.c_int64),
                                               C.c_void_p, C.c_void_p, C.c_void_p]
        lib.ref_write_matrix_market.argtypes = [C.c_char_p, C.c_int64, _i64p, _i32p, _f64p]
        lib.ref_spmv_traffic_bytes.restype = C.c_double
        lib.ref_spmv_traffic_bytes.argtypes = [C.c_int64, C.c_int64, C.c_int]
        lib.ref_solve.argtypes = [C.c_int, C.c_int64, _i64p, _i32p, _f64p, C.c_int, _f64p, _f64p,
                                  C.c_double, C.c_int, C.c_int, C.c_int, C.POINTER(C.c_int),
                                  C.POINTER(C.c_double)]
        _ref = lib
    return _ref


class Csr:
    """Host CSR held as numpy arrays (int64 offsets, int32 cols, fp64 vals)."""

    def __init__(self, n, off, col, val):
        self.n = int(n)
        self.off = np.ascontiguousarray(off, dtype=np.int64)
        self.col = np.ascontiguousarray(col, dtype=np.int32)
        self.val = np.ascontiguousarray(val, dtype=np.float64)

    @property
    def nnz(self) -> int:
        return int(self.off[-1])

    def _orc(self) -> OrcCsr:
        s = OrcCsr()
        s.n = self.n
        s.nnz = self.nnz
        s.off = self.off.ctypes.data_as(C.POINTER(C.c_int64))
        s.col = self.col.ctypes.data_as(C.POINTER(C.c_int32))
        s.val = self.val.ctypes.data_as(C.POINTER(C.c_double))
        return s

    def to_scipy(self):
        import scipy.sparse as sp
        return sp.csr_matrix((self.val, self.col, self.off), shape=(self.n, self.n))


def _from_orc(s: OrcCsr) -> Csr:
    n, nnz = s.n, s.nnz
    off = np.ctypeslib.as_array(s.off, shape=(n + 1,)).copy()
    col = np.ctypeslib.as_array(s.col, shape=(nnz,)).copy() if nnz else np.zeros(0, np.int32)
    val = np.ctypeslib.as_array(s.val, shape=(nnz,)).copy() if nnz else np.zeros(0)
    orc().orc_csr_free(C.byref(s))
    return Csr(n, off, col, val)


STENCIL_KINDS = {"poisson7": 0, "convdiff7": 1, "stencil27": 2, "poisson5": 3}


def gen_stencil(kind: str, nx: int, ny: int, nz: int, seed: int = 0) -> Csr:
    s = OrcCsr()
    rc = orc().orc_gen_stencil(STENCIL_KINDS[kind], nx, ny, nz, seed, C.byref(s))
    assert rc == 0, rc
    return _from_orc(s)


def gen_banded(n: int, band: int, kmin: int, kmax: int, seed: int) -> Csr:
    s = OrcCsr()
    rc = orc().orc_gen_banded(n, band, kmin, kmax, seed, C.byref(s))
    assert rc == 0, rc
    return _from_orc(s)


def rhs(n: int, m: int, seed: int) -> np.ndarray:
    b = np.empty(n * m)
    orc().orc_rhs(n, m, seed, b)
    return b


def spmv(a: Csr, x: np.ndarray, m: int) -> np.ndarray:
    y = np.empty(a.n * m)
    s = a._orc()
    orc().orc_spmv(C.byref(s), m, np.ascontiguousarray(x, dtype=np.float64), y)
    return y


def spmv_transpose(a: Csr, x: np.ndarray, m: int) -> np.ndarray:
    y = np.empty(a.n * m)
    s = a._orc()
    orc().orc_spmv_transpose(C.byref(s), m, np.ascontiguousarray(x, dtype=np.float64), y)
    return y


def dot_exact(a: np.ndarray, b: np.ndarray, m: int) -> np.ndarray:
    out = np.empty(m)
    n = a.size // m
    orc().orc_dot_exact(n, m, np.ascontiguousarray(a), np.ascontiguousarray(b), out)
    return out


def sum_exact(v: np.ndarray) -> float:
    v = np.ascontiguousarray(v, dtype=np.float64)
    return orc().orc_sum_exact(v.size, v)


def update(n: int, m: int, terms, out: np.ndarray) -> None:
    """out = sum coeff_t * src_t (acc from 0.0, terms in order)."""
    nt = len(terms)
    cs = (C.c_void_p * nt)(*[np.ascontiguousarray(c).ctypes.data for c, _ in terms])
    vs = (C.c_void_p * nt)(*[v.ctypes.data for _, v in terms])
    keep = [c for c, _ in terms]  # noqa: F841 keep arrays alive
    orc().orc_update(n, m, nt, cs, vs, out)


def preconditioned(method: str) -> bool:
    return bool(orc().orc_method_preconditioned(METHODS[method]))


def solve(a: Csr, b: np.ndarray, m: int, method="bicgstab", formulation="merged", tol=1e-8,
          fixed=False, maxit=1000, x0=None, precond_alpha=None):
    """precond_alpha None: identity (2) for the preconditioned methods, else none."""
    x = np.zeros(a.n * m) if x0 is None else np.array(x0, dtype=np.float64)
    hist = np.full((maxit + 1) * m, np.nan)
    rep = OrcReport()
    s = a._orc()
    pa = (2 if preconditioned(method) else 0) if precond_alpha is None else precond_alpha
    rc = orc().orc_solve_pc(C.byref(s), m, np.ascontiguousarray(b), x, METHODS[method],
                            FORMULATIONS[formulation], pa, tol, int(bool(fixed)), maxit, hist, C.byref(rep))
    assert rc == 0, rc
    its = rep.iterations
    return {
        "x": x,
        "hist": hist.reshape(maxit + 1, m)[: its + 1].copy(),
        "iterations": its,
        "converged": bool(rep.converged),
        "breakdown": rep.breakdown,
        "breakdown_iter": rep.breakdown_iter,
        "breakdown_col": rep.breakdown_col,
    }


# ---- reference kernels ---------------------------------------------------
def ref_gen_poisson_7pt(nx, ny, nz) -> Csr:
    lib = ref()
    nnz = C.c_int64()
    assert lib.ref_gen_poisson_7pt(nx, ny, nz, C.byref(nnz), None, None, None) == 0
    n = nx * ny * nz
    off = np.empty(n + 1, np.int64)
    col = np.empty(nnz.value, np.int32)
    val = np.empty(nnz.value)
    assert lib.ref_gen_poisson_7pt(nx, ny, nz, C.byref(nnz), off.ctypes.data, col.ctypes.data,
                                   val.ctypes.data) == 0
    return Csr(n, off, col, val)


def ref_gen_poisson_5pt(nx, ny) -> Csr:
    lib = ref()
    nnz = C.c_int64()
    assert lib.ref_gen_poisson_5pt(nx, ny, C.byref(nnz), None, None, None) == 0
    n = nx * ny
    off = np.empty(n + 1, np.int64)
    col = np.empty(nnz.value, np.int32)
    val = np.empty(nnz.value)
    assert lib.ref_gen_poisson_5pt(nx, ny, C.byref(nnz), off.ctypes.data, col.ctypes.data, val.ctypes.data) == 0
    return Csr(n, off, col, val)


def ref_spmv(a: Csr, x: np.ndarray, m: int, threads: int = 1) -> np.ndarray:
    y = np.empty(a.n * m)
    rc = ref().ref_spmv(a.n, a.off, a.col, a.val, m, np.ascontiguousarray(x), y, threads)
    assert rc == 0, ref().ref_last_error()
    return y


def ref_spmv_transpose(a: Csr, x: np.ndarray, m: int) -> np.ndarray:
    y = np.empty(a.n * m)
    rc = ref().ref_spmv_transpose(a.n, a.off, a.col, a.val, m, np.ascontiguousarray(x), y)
    assert rc == 0, ref().ref_last_error()
    return y


def ref_read_matrix_market(path):
    """core::read_matrix_market from the reference sources: Csr or raises RuntimeError(msg)."""
    lib = ref()
    n, nnz = C.c_int64(), C.c_int64()
    if lib.ref_read_matrix_market(str(path).encode(), C.byref(n), C.byref(nnz), None, None, None):
        raise RuntimeError(lib.ref_last_error().decode())
    off = np.empty(n.value + 1, np.int64)
    col = np.empty(nnz.value, np.int32)
    val = np.empty(nnz.value)
    assert lib.ref_read_matrix_market(str(path).encode(), C.byref(n), C.byref(nnz), off.ctypes.data,
                                      col.ctypes.data, val.ctypes.data) == 0
    return Csr(n.value, off, col, val)


def ref_solve_hist(a: Csr, b: np.ndarray, m: int, method="bicgstab", tol=1e-8, fixed=False, maxit=1000,
                   threads=1):
    """ref_solve plus its relative residual history ((iterations+1) x m)."""
    lib = ref()
    if not getattr(lib, "_hist_bound", False):
        lib.ref_solve_hist.argtypes = [C.c_int, C.c_int64, _i64p, _i32p, _f64p, C.c_int, _f64p, _f64p,
                                       C.c_double, C.c_int, C.c_int, C.c_int, C.POINTER(C.c_int),
                                       C.POINTER(C.c_double), _f64p]
        lib.ref_solve_hist.restype = C.c_int
        lib._hist_bound = True
    x = np.zeros(a.n * m)
    hist = np.full((maxit + 1) * m, np.nan)
    its = C.c_int()
    secs = C.c_double()
    rc = lib.ref_solve_hist(METHODS[method], a.n, a.off, a.col, a.val, m, np.ascontiguousarray(b), x, tol,
                            int(bool(fixed)), maxit, threads, C.byref(its), C.byref(secs), hist)
    assert rc == 0, lib.ref_last_error()
    return x, its.value, hist.reshape(maxit + 1, m)[: its.value + 1].copy()


def ref_write_matrix_market(a: Csr, path) -> None:
    assert ref().ref_write_matrix_market(str(path).encode(), a.n, a.off, a.col, a.val) == 0


def ref_solve(a: Csr, b: np.ndarray, m: int, method="bicgstab", tol=1e-8, fixed=False, maxit=1000,
              threads=None, timing=False):
    """Restated merged solver on the reference's own kernels (naive dots).

    Returns (x, iterations) or, with timing=True, (x, iterations, loop_seconds)."""
    threads = threads or os.cpu_count() or 1
    x = np.zeros(a.n * m)
    its = C.c_int()
    secs = C.c_double()
    rc = ref().ref_solve(METHODS[method], a.n, a.off, a.col, a.val, m, np.ascontiguousarray(b), x,
                         tol, int(bool(fixed)), maxit, threads, C.byref(its), C.byref(secs))
    assert rc == 0, ref().ref_last_error()
    return (x, its.value, secs.value) if timing else (x, its.value)
