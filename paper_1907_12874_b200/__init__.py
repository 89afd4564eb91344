"""B200-native multi-RHS BiCGStab hot path (arXiv:1907.12874).

Python mirror of the reference's operator interface for this path, over the
C ABI in ``include/mbstab_b200.h``:

=========================  ==============================================
this module                reference (``/root/reference/proj``)
=========================  ==============================================
``CsrMatrix``              ``core::CsrMatrix`` (csr.hpp:13-30)
``CsrMatrix.validate``     ``CsrMatrix::validate`` (csr.cpp:8-32)
``Context.upload``         (device copy of a ``CsrMatrix``)
``MultiVector``            ``core::MultiVector`` (types.hpp:13-35)
``spmv``                   ``core::spmv`` (spmv.hpp:16-17)
``spmv_traffic_bytes``     ``core::spmv_traffic_bytes`` (spmv.cpp:10-16)
``UpdateStatement`` ...    ``kernels::Statement`` family (statement.hpp:13-45)
``analyze_traffic``        ``kernels::analyze_traffic`` (statement.hpp:65)
``split_basic_traffic``    ``kernels::split_basic`` + analyze (statement.hpp:73)
``execute_group``          ``kernels::execute_group`` (execute.hpp:26-30)
``solve``                  ``solvers::solve`` (missing in proj/)
``method_schedule``        ``solvers::method_schedule``
``gen_poisson_7pt``        ``core::gen_poisson_7pt`` (generators.cpp:37-67)
=========================  ==============================================

Errors follow the reference: API misuse raises ``ValueError`` (the
reference's ``std::invalid_argument``), CUDA/NCCL failures ``RuntimeError``,
solver breakdown ``BreakdownError``.  All compute runs in the CUDA library;
there is no CPU fallback.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import Sequence

import numpy as np

from ._lib import BreakdownError, MbgReport, MbgStatement, build, check, lib  # noqa: F401

METHODS = {"bicgstab": 0, "rbicgstab": 1, "pipebicgstab": 2, "ibicgstab": 3, "pbicgstab": 4,
           "ppipebicgstab": 5}
# these take (and require) a preconditioner M^-1
PRECONDITIONED = ("rbicgstab", "pbicgstab", "ppipebicgstab")
FORMULATIONS = {"merged": 0, "basic": 1, "fused": 2}


def _ptr(a: np.ndarray) -> int:
    return a.ctypes.data


# ---------------------------------------------------------------------------
# host containers
# ---------------------------------------------------------------------------
class CsrMatrix:
    """Square CSR (offsets int64[n+1], cols int32[nnz], vals fp64[nnz])."""

    def __init__(self, n_rows: int, row_offsets, col_indices, values):
        self.n_rows = int(n_rows)
        self.row_offsets = np.ascontiguousarray(row_offsets, dtype=np.int64)
        self.col_indices = np.ascontiguousarray(col_indices, dtype=np.int32)
        self.values = np.ascontiguousarray(values, dtype=np.float64)

    def nnz(self) -> int:
        return int(self.row_offsets[-1]) if self.row_offsets.size else 0

    def avg_row_nnz(self) -> float:
        return self.nnz() / self.n_rows if self.n_rows else 0.0

    def validate(self) -> None:
        if self.row_offsets.size != self.n_rows + 1:
            raise ValueError("csr: row_offsets length must be n_rows+1")
        if self.col_indices.size != self.values.size:
            raise ValueError("csr: col_indices and values length mismatch")
        check(lib().mbg_csr_validate(self.n_rows, _ptr(self.row_offsets), _ptr(self.col_indices),
                                     self.col_indices.size))


def gen_stencil(kind: str, nx: int, ny: int, nz: int, seed: int = 0) -> CsrMatrix:
    """kind: 'poisson7' (gen_poisson_7pt), 'convdiff7' or 'stencil27' (BASELINE configs)."""
    k = {"poisson7": 0, "convdiff7": 1, "stencil27": 2, "poisson5": 3}[kind]
    n = nx * ny * nz
    nnz = C.c_int64()
    off = np.empty(n + 1, np.int64)
    check(lib().mbg_gen_stencil(k, nx, ny, nz, seed, C.byref(nnz), _ptr(off), None, None))
    col = np.empty(nnz.value, np.int32)
    val = np.empty(nnz.value, np.float64)
    check(lib().mbg_gen_stencil(k, nx, ny, nz, seed, C.byref(nnz), _ptr(off), _ptr(col), _ptr(val)))
    return CsrMatrix(n, off, col, val)


def gen_poisson_7pt(nx: int, ny: int, nz: int) -> CsrMatrix:
    return gen_stencil("poisson7", nx, ny, nz)


def gen_poisson_5pt(nx: int, ny: int) -> CsrMatrix:
    """core::gen_poisson_5pt (generators.cpp:69-91): 2-D, diagonal 4, neighbours -1."""
    return gen_stencil("poisson5", nx, ny, 1)


def gen_banded(n: int, band: int = 65536, kmin: int = 16, kmax: int = 32, seed: int = 4) -> CsrMatrix:
    nnz = C.c_int64()
    off = np.empty(n + 1, np.int64)
    check(lib().mbg_gen_banded(n, band, kmin, kmax, seed, C.byref(nnz), _ptr(off), None, None))
    col = np.empty(nnz.value, np.int32)
    val = np.empty(nnz.value, np.float64)
    check(lib().mbg_gen_banded(n, band, kmin, kmax, seed, C.byref(nnz), _ptr(off), _ptr(col), _ptr(val)))
    return CsrMatrix(n, off, col, val)


def gen_rhs(n: int, m: int, seed: int) -> np.ndarray:
    b = np.empty(n * m, np.float64)
    check(lib().mbg_gen_rhs(n, m, seed, _ptr(b)))
    return b


# BASELINE.json configs
CONFIGS = {
    1: dict(matrix=("poisson7", 32, 32, 32), m=1, seed=0, method="bicgstab", tol=1e-8, maxit=1000, fixed=False),
    2: dict(matrix=("convdiff7", 128, 128, 128), m=8, seed=1, method="bicgstab", tol=1e-8, maxit=1000,
            fixed=False),
    3: dict(matrix=("stencil27", 192, 192, 192), m=16, seed=2, method="rbicgstab", tol=1e-8, maxit=1000,
            fixed=False),
    4: dict(matrix=("convdiff7", 320, 320, 320), m=32, seed=3, method="pipebicgstab", tol=1e-8, maxit=200,
            fixed=True),
    5: dict(matrix=("banded", 8_000_000), m=8, seed=4, method="bicgstab", tol=1e-8, maxit=100, fixed=True),
}


def config_matrix(cfg: dict, seed: int | None = None) -> CsrMatrix:
    kind = cfg["matrix"][0]
    s = cfg["seed"] if seed is None else seed
    if kind == "banded":
        return gen_banded(cfg["matrix"][1], 65536, 16, 32, s)
    return gen_stencil(kind, *cfg["matrix"][1:], seed=s)


# ---------------------------------------------------------------------------
# device objects
# ---------------------------------------------------------------------------
class Context:
    """One CUDA device with its streams (and optional NCCL communicator)."""

    def __init__(self, device: int = 0):
        h = C.c_void_p()
        check(lib().mbg_ctx_create(device, C.byref(h)))
        self.h = h
        self.device = device

    def close(self) -> None:
        if self.h:
            check(lib().mbg_ctx_destroy(self.h))
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def synchronize(self) -> None:
        check(lib().mbg_ctx_synchronize(self.h))

    def set_small_path(self, enable: bool) -> None:
        """Small classical solves in one cooperative launch (default on)."""
        check(lib().mbg_ctx_set_small_path(self.h, int(bool(enable))))

    def reserve_sms(self, count: int) -> None:
        """Size the persistent grids for (device SMs - count) SMs (bitwise-neutral)."""
        check(lib().mbg_ctx_reserve_sms(self.h, int(count)))

    def launches(self) -> int:
        return int(lib().mbg_ctx_launches(self.h))

    def init_comm(self, rank: int, world: int, nccl_id: bytes) -> None:
        check(lib().mbg_ctx_init_comm(self.h, rank, world, nccl_id))

    def upload(self, a: CsrMatrix, parts: Sequence[int] | None = None, my_part: int = 0,
               any_order: bool = False) -> "DeviceCsr":
        return DeviceCsr(self, a, parts, my_part, any_order)

    def multivector(self, n: int, m: int, data: np.ndarray | None = None) -> "MultiVector":
        v = MultiVector(self, n, m)
        if data is not None:
            v.upload(data)
        return v


def local_group(ctxs: Sequence["Context"]) -> None:
    """Validation only: emulate a len(ctxs)-rank communicator on one GPU."""
    arr = (C.c_void_p * len(ctxs))(*[c.h for c in ctxs])
    check(lib().mbg_local_group_create(arr, len(ctxs)))


def comm_unique_id() -> bytes:
    buf = C.create_string_buffer(128)
    check(lib().mbg_comm_unique_id(buf))
    return buf.raw


class DeviceCsr:
    def __init__(self, ctx: Context, a: CsrMatrix, parts=None, my_part: int = 0, any_order: bool = False):
        self.ctx = ctx
        h = C.c_void_p()
        if parts is None:
            up = lib().mbg_csr_upload_any_order if any_order else lib().mbg_csr_upload
            check(up(ctx.h, a.n_rows, _ptr(a.row_offsets), _ptr(a.col_indices), _ptr(a.values), C.byref(h)))
            self.row_begin, self.row_end = 0, a.n_rows
        else:
            b = np.ascontiguousarray(parts, dtype=np.int64)
            check(lib().mbg_csr_upload_partitioned(ctx.h, a.n_rows, _ptr(a.row_offsets), _ptr(a.col_indices),
                                                   _ptr(a.values), b.size - 1, _ptr(b), my_part, C.byref(h)))
            self.row_begin, self.row_end = int(b[my_part]), int(b[my_part + 1])
        self.h = h
        self.n_global = a.n_rows
        self.n = int(lib().mbg_csr_rows(h))
        self.nnz = int(lib().mbg_csr_nnz(h))

    def set_grid(self, nx: int, ny: int, nz: int) -> bool:
        """Structured-grid hint: a grid-neighbour operator gets a stencil twin
        (implicit columns, TMA-staged x planes; m in {4, 8, 16, 32}) and long-row
        stencils a brick-reordered twin for the other m (bitwise-identical
        results).  Returns True if reordered."""
        check(lib().mbg_csr_set_grid(self.ctx.h, self.h, nx, ny, nz))
        return bool(lib().mbg_csr_reordered(self.h))

    def clear_grid(self) -> None:
        """Drop the stencil twin (detected at upload or set by set_grid): the
        SpMM takes the CSR path (A/B measurements)."""
        check(lib().mbg_csr_clear_grid(self.h))

    @property
    def stencil_kind(self) -> int:
        """7 or 27 when the stencil twin is in place, else 0."""
        return int(lib().mbg_csr_stencil_kind(self.h))

    def stage_info(self):
        """(staged, reuse): whether the gather-once SpMM tiling is in use."""
        st, ru = C.c_int(0), C.c_double(0.0)
        check(lib().mbg_csr_stage_info(self.h, C.byref(st), C.byref(ru)))
        return bool(st.value), float(ru.value)

    def sort_info(self):
        """(sorted, lane_efficiency): whether the CSR SpMM walks the
        length-sorted twin, and the natural order's useful share of gather slots."""
        so, ef = C.c_int(0), C.c_double(0.0)
        check(lib().mbg_csr_sort_info(self.h, C.byref(so), C.byref(ef)))
        return bool(so.value), float(ef.value)

    def __del__(self):
        try:
            if self.h:
                lib().mbg_csr_free(self.h)
                self.h = None
        except Exception:
            pass


class MultiVector:
    """n x m fp64 block on the device, row-interleaved (element (i,c) at i*m+c)."""

    def __init__(self, ctx: Context, n: int, m: int):
        self.ctx = ctx
        h = C.c_void_p()
        check(lib().mbg_mv_alloc(ctx.h, n, m, C.byref(h)))
        self.h = h
        self.n_rows, self.n_cols = int(n), int(m)

    def __del__(self):
        try:
            if self.h:
                lib().mbg_mv_free(self.h)
                self.h = None
        except Exception:
            pass

    def upload(self, data: np.ndarray) -> None:
        d = np.ascontiguousarray(data, dtype=np.float64).reshape(-1)
        if d.size != self.n_rows * self.n_cols:
            raise ValueError("multivector: size mismatch")
        check(lib().mbg_mv_upload(self.h, _ptr(d)))

    def download(self) -> np.ndarray:
        out = np.empty(self.n_rows * self.n_cols, np.float64)
        check(lib().mbg_mv_download(self.h, _ptr(out)))
        return out

    def fill(self, value: float) -> None:
        check(lib().mbg_mv_fill(self.h, value))


# ---------------------------------------------------------------------------
# operators
# ---------------------------------------------------------------------------
def debug_guard_check() -> int:
    """Checked builds (MBG_CHECKED=1): damaged guard zones found so far (0 = none)."""
    v = C.c_int64(0)
    rc = lib().mbg_debug_guard_check(C.byref(v))
    if rc != 0 and v.value == 0:
        check(rc)
    return int(v.value)


def debug_write_past_end(v: "MultiVector") -> None:
    """Checked builds: write one double past v's allocation (tests the guards)."""
    check(lib().mbg_debug_write_past_end(v.h))


def spmv(ctx: Context, a: DeviceCsr, x: MultiVector, y: MultiVector) -> None:
    """y = A x (core::spmv).  Raises ValueError on shape mismatch or x is y."""
    check(lib().mbg_spmv(ctx.h, a.h, x.h, y.h))


def true_residual(ctx: Context, a: DeviceCsr, b: MultiVector, x: MultiVector) -> np.ndarray:
    """||b - A x||_2 / ||b||_2 per column (exact dots)."""
    out = np.empty(b.n_cols)
    check(lib().mbg_true_residual(ctx.h, a.h, b.h, x.h, _ptr(out)))
    return out


def spmv_transpose(ctx: Context, a: DeviceCsr, x: MultiVector, y: MultiVector) -> None:
    """core::spmv_transpose: y = A^T x in the reference's serial summation order."""
    check(lib().mbg_spmv_transpose(ctx.h, a.h, x.h, y.h))


def spmv_traffic_bytes(n: int, nnz: int, m: int) -> float:
    return float(lib().mbg_spmv_traffic_bytes(n, nnz, m))


def spmv_compulsory_bytes(n: int, nnz: int, m: int) -> float:
    return float(lib().mbg_spmv_compulsory_bytes(n, nnz, m))


@dataclass
class UpdateStatement:
    """out(i,c) = sum_t coeff_t[c] * vec_t(i,c)   (statement.hpp:22-28)."""
    out: int
    terms: list = field(default_factory=list)   # [(coeff array (m,), vector id)]


@dataclass
class DotStatement:
    """slot[c] = sum_i left(i,c) * right(i,c)   (statement.hpp:30-36)."""
    left: int
    right: int
    slot: int


def _statements(group, keep: list):
    arr = (MbgStatement * max(1, len(group)))()
    for i, st in enumerate(group):
        s = arr[i]
        if isinstance(st, UpdateStatement):
            if len(st.terms) > 8:
                raise ValueError("execute_group: too many terms")
            s.kind, s.out, s.nterms = 0, st.out, len(st.terms)
            for t, (coeff, vec) in enumerate(st.terms):
                c = np.ascontiguousarray(coeff, dtype=np.float64)
                keep.append(c)
                s.term_vec[t] = vec
                s.term_coeff[t] = c.ctypes.data
        elif isinstance(st, DotStatement):
            s.kind, s.left, s.right, s.slot = 1, st.left, st.right, st.slot
        else:
            raise ValueError("statement group: unknown statement")
    return arr


def analyze_traffic(group) -> tuple[int, int]:
    keep: list = []
    arr = _statements(group, keep)
    r, w = C.c_int(), C.c_int()
    check(lib().mbg_analyze_traffic(arr, len(group), C.byref(r), C.byref(w)))
    return r.value, w.value


def split_basic_traffic(group, first_temp_id: int = 100) -> tuple[int, int, int]:
    keep: list = []
    arr = _statements(group, keep)
    r, w, g = C.c_int(), C.c_int(), C.c_int()
    check(lib().mbg_split_basic_traffic(arr, len(group), first_temp_id, C.byref(r), C.byref(w), C.byref(g)))
    return r.value, w.value, g.value


def execute_group(ctx: Context, group, vectors: Sequence[MultiVector], nslots: int | None = None) -> np.ndarray:
    """Fused single-pass execution; returns dot results (nslots, m), exact."""
    keep: list = []
    arr = _statements(group, keep)
    if nslots is None:
        nslots = 1 + max([st.slot for st in group if isinstance(st, DotStatement)], default=-1)
    m = vectors[0].n_cols if vectors else 1
    out = np.zeros(max(1, nslots) * m)
    handles = (C.c_void_p * max(1, len(vectors)))(*[v.h if v is not None else None for v in vectors])
    check(lib().mbg_execute_group(ctx.h, arr, len(group), handles, len(vectors), _ptr(out), nslots))
    return out[: nslots * m].reshape(nslots, m)


def method_schedule(method: str, formulation: str = "merged") -> dict:
    r, w, s, k = C.c_int(), C.c_int(), C.c_int(), C.c_int()
    dots = (C.c_int * 8)()
    check(lib().mbg_method_schedule(METHODS[method], FORMULATIONS[formulation], C.byref(r), C.byref(w),
                                    C.byref(s), C.byref(k), dots))
    return {"reads": r.value, "writes": w.value, "spmvs": s.value, "reductions": list(dots[: min(k.value, 8)])}


def method_schedule_pc(method: str, formulation: str = "merged", precond_alpha: int | None = None) -> dict:
    """SPEC.md:236-244 form: vector transfers without the preconditioner, plus
    the M^-1 applications per iteration (each worth precond_alpha transfers)."""
    pa = (2 if method in PRECONDITIONED else 0) if precond_alpha is None else precond_alpha
    r, w, s, ap, k = C.c_int(), C.c_int(), C.c_int(), C.c_int(), C.c_int()
    dots = (C.c_int * 8)()
    check(lib().mbg_method_schedule_pc(METHODS[method], FORMULATIONS[formulation], pa, C.byref(r), C.byref(w),
                                       C.byref(s), C.byref(ap), C.byref(k), dots))
    return {"vec": r.value + w.value, "reads": r.value, "writes": w.value, "spmvs": s.value,
            "precond": ap.value, "reductions": list(dots[: min(k.value, 8)])}


@dataclass
class SolveReport:
    iterations: int
    converged: bool
    breakdown: int
    breakdown_iter: int
    breakdown_col: int
    residual_history: np.ndarray          # (iterations+1, m) relative recursive residuals
    vector_reads: int
    vector_writes: int
    spmv_bytes: float
    compulsory_bytes: float
    reductions: int
    gpu_launches: int
    loop_ms: float


def _report(rep: MbgReport, hist: np.ndarray | None, m: int, maxit: int) -> SolveReport:
    h = None
    if hist is not None:
        h = hist.reshape(maxit + 1, m)[: rep.iterations + 1].copy()
    return SolveReport(rep.iterations, bool(rep.converged), rep.breakdown, rep.breakdown_iter, rep.breakdown_col,
                       h, rep.vector_reads, rep.vector_writes, rep.spmv_bytes, rep.compulsory_bytes,
                       rep.reductions, rep.gpu_launches, rep.loop_ms)


def solve(ctx: Context, a: DeviceCsr, b: MultiVector, x: MultiVector, method: str = "bicgstab",
          formulation: str = "merged", tol: float = 1e-8, fixed: bool = False, max_iters: int = 1000,
          history: bool = True, precond_alpha: int | None = None) -> SolveReport:
    """Device-resident solve; x holds x0 on entry and the solution on exit.

    precond_alpha: None = identity M^-1 for the preconditioned methods (none
    otherwise); 2 = identity; even >= 4 = synthetic(alpha)."""
    m = b.n_cols
    hist = np.full((max_iters + 1) * m, np.nan) if history else None
    rep = MbgReport()
    if precond_alpha is None:
        rc = lib().mbg_solve(ctx.h, a.h, b.h, x.h, METHODS[method], FORMULATIONS[formulation], tol,
                             int(bool(fixed)), max_iters, _ptr(hist) if hist is not None else None, C.byref(rep))
    else:
        rc = lib().mbg_solve_pc(ctx.h, a.h, b.h, x.h, METHODS[method], FORMULATIONS[formulation],
                                int(precond_alpha), tol, int(bool(fixed)), max_iters,
                                _ptr(hist) if hist is not None else None, C.byref(rep))
    check(rc)
    return _report(rep, hist, m, max_iters)


def solve_profile(ctx: Context, a: DeviceCsr, b: MultiVector, x: MultiVector, method: str = "bicgstab",
                  formulation: str = "merged", tol: float = 1e-8, fixed: bool = False,
                  max_iters: int = 1000) -> tuple[SolveReport, dict]:
    """Solve once with CUDA events around every kernel of the loop.

    Returns (report, {label: (launches, total_ms, algorithmic bytes per launch)})."""
    import json
    buf = C.create_string_buffer(1 << 16)
    rep = MbgReport()
    check(lib().mbg_solve_profile(ctx.h, a.h, b.h, x.h, METHODS[method], FORMULATIONS[formulation], tol,
                                  int(bool(fixed)), max_iters, buf, len(buf), C.byref(rep)))
    return _report(rep, None, b.n_cols, max_iters), json.loads(buf.value.decode())


def solve_host(ctx: Context, a: DeviceCsr, b: np.ndarray, x: np.ndarray, m: int, method: str = "bicgstab",
               formulation: str = "merged", tol: float = 1e-8, fixed: bool = False, max_iters: int = 1000,
               history: bool = True) -> SolveReport:
    """End-to-end solve from HOST buffers: b, x0 uploaded, x downloaded in place."""
    if not (b.flags.c_contiguous and x.flags.c_contiguous and b.dtype == np.float64 and x.dtype == np.float64):
        raise ValueError("solve_host: b and x must be C-contiguous float64")
    hist = np.full((max_iters + 1) * m, np.nan) if history else None
    rep = MbgReport()
    rc = lib().mbg_solve_host(ctx.h, a.h, m, _ptr(b), _ptr(x), METHODS[method], FORMULATIONS[formulation], tol,
                              int(bool(fixed)), max_iters, _ptr(hist) if hist is not None else None, C.byref(rep))
    check(rc)
    return _report(rep, hist, m, max_iters)


# ---------------------------------------------------------------------------
# partition / exact-dot host hooks (used by the multi-rank CPU tests)
# ---------------------------------------------------------------------------
def infer_grid(a: CsrMatrix) -> tuple[int, int, int]:
    """Host-only: the (nx, ny, nz) the upload would try for a lexicographic 7- /
    27-point grid operator, (0, 0, 0) when the matrix does not look like one."""
    nx, ny, nz = C.c_int(0), C.c_int(0), C.c_int(0)
    check(lib().mbg_infer_grid(a.n_rows, _ptr(a.row_offsets), _ptr(a.col_indices), C.byref(nx), C.byref(ny),
                               C.byref(nz)))
    return nx.value, ny.value, nz.value


def sorted_twin_plan(row_offsets, window: int = 4096) -> dict:
    """Host-only plan of the CSR SpMM's length-sorted twin: the row stored in
    each slot (-1 = padding), the groups' first batches, the tile list and the
    natural order's lane efficiency."""
    off = np.ascontiguousarray(row_offsets, dtype=np.int64)
    n = off.size - 1
    eff, nt, ns = C.c_double(0.0), C.c_int64(0), C.c_int64(0)
    check(lib().mbg_sorted_twin_plan(n, _ptr(off), window, C.byref(ns), None, C.byref(eff), C.byref(nt), None, None))
    rowid = np.empty(max(1, ns.value), np.int32)
    tiles = np.empty(max(1, 4 * nt.value), np.int32)
    goff = np.empty(n // 8 + 2, np.int32)
    check(lib().mbg_sorted_twin_plan(n, _ptr(off), window, None, _ptr(rowid), None, None, _ptr(tiles), _ptr(goff)))
    return {"rowid": rowid[: ns.value].copy(), "tiles": tiles[: 4 * nt.value].reshape(-1, 4).copy(),
            "group_off": goff, "lane_efficiency": float(eff.value)}


def halo_plan(a: CsrMatrix, bounds: Sequence[int], my_part: int, transpose: bool = False) -> dict:
    """Host-only halo plan of part `my_part` (of A^T when transpose=True)."""
    L = lib()
    fn = L.mbg_transpose_halo_plan if transpose else L.mbg_halo_plan
    b = np.ascontiguousarray(bounds, dtype=np.int64)
    n_own, n_halo, nnz, npeers = C.c_int64(), C.c_int64(), C.c_int64(), C.c_int()
    args0 = [a.n_rows, _ptr(a.row_offsets), _ptr(a.col_indices), _ptr(a.values), b.size - 1, _ptr(b), my_part,
             C.byref(n_own), C.byref(n_halo), C.byref(nnz)]
    check(fn(*args0, None, None, None, None, C.byref(npeers), None, None, None, None, None))
    off = np.empty(n_own.value + 1, np.int32)
    col = np.empty(nnz.value, np.int32)
    val = np.empty(nnz.value, np.float64)
    hg = np.empty(max(1, n_halo.value), np.int64)
    pp = np.empty(max(1, npeers.value), np.int32)
    psc = np.empty(max(1, npeers.value), np.int64)
    pro = np.empty(max(1, npeers.value), np.int64)
    prc = np.empty(max(1, npeers.value), np.int64)
    # send rows: at most n_own per peer
    psr = np.empty(max(1, npeers.value * max(1, n_own.value)), np.int32)
    check(fn(*args0, _ptr(off), _ptr(col), _ptr(val), _ptr(hg), C.byref(npeers), _ptr(pp), _ptr(psc),
             _ptr(psr), _ptr(pro), _ptr(prc)))
    peers, so = [], 0
    for i in range(npeers.value):
        cnt = int(psc[i])
        peers.append({"part": int(pp[i]), "send_rows": psr[so:so + cnt].copy(), "recv_offset": int(pro[i]),
                      "recv_count": int(prc[i])})
        so += cnt
    return {"n_own": n_own.value, "n_halo": n_halo.value, "off": off, "col": col, "val": val,
            "halo_global": hg[: n_halo.value].copy(), "peers": peers}


def exact_slot_words() -> int:
    return int(lib().mbg_exact_slot_words())


def exact_accumulate(a: np.ndarray, b: np.ndarray, m: int, digits: np.ndarray | None = None) -> np.ndarray:
    w = exact_slot_words()
    if digits is None:
        digits = np.zeros(m * w, np.int64)
    a = np.ascontiguousarray(a, np.float64)
    b = np.ascontiguousarray(b, np.float64)
    check(lib().mbg_exact_accumulate_host(a.size // m, m, _ptr(a), _ptr(b), _ptr(digits)))
    return digits


def exact_round(digits: np.ndarray, count: int) -> np.ndarray:
    out = np.empty(count)
    d = np.ascontiguousarray(digits, np.int64)
    check(lib().mbg_exact_round_host(_ptr(d), count, _ptr(out)))
    return out


# ---- MatrixMarket (core::read_matrix_market / write_matrix_market) ----------
def read_matrix_market(path) -> CsrMatrix:
    """Coordinate real/integer, general/symmetric MatrixMarket file -> CsrMatrix
    (matrix_market.cpp:38-113 contract; RuntimeError "<name>:<line>: message")."""
    h = C.c_void_p()
    n, nnz = C.c_int64(), C.c_int64()
    check(lib().mbg_mm_read(str(path).encode(), C.byref(h), C.byref(n), C.byref(nnz)))
    try:
        off = np.empty(n.value + 1, np.int64)
        col = np.empty(nnz.value, np.int32)
        val = np.empty(nnz.value, np.float64)
        check(lib().mbg_mm_copy(h, _ptr(off), _ptr(col), _ptr(val)))
    finally:
        lib().mbg_mm_free(h)
    return CsrMatrix(int(n.value), off, col, val)


def write_matrix_market(a: CsrMatrix, path) -> None:
    check(lib().mbg_mm_write(str(path).encode(), a.n_rows, _ptr(a.row_offsets), _ptr(a.col_indices),
                             _ptr(a.values)))


def fusion_bench(ctx: Context, n: int = 100_000_000, reps: int = 10) -> dict:
    """Fig. 2 runs #1-#3: ms and GB/s per run, run1/run2
    ratio (paper: ~1.76, memory-traffic ratio 1.8, flop ratio 1.5), and whether
    run #3 reproduced run #1 bit for bit."""
    ms = np.zeros(3)
    gbs = np.zeros(3)
    same = C.c_int(0)
    check(lib().mbg_fusion_bench(ctx.h, n, reps, _ptr(ms), _ptr(gbs), C.byref(same)))
    return {"n": n, "reps": reps, "ms": ms.tolist(), "GBps": gbs.tolist(),
            "run1_over_run2": float(ms[0] / ms[1]), "run3_over_run2": float(ms[2] / ms[1]),
            "run3_equals_run1": bool(same.value)}


class _PinnedBlock:
    def __init__(self, nbytes: int):
        self.ptr = C.c_void_p()
        check(lib().mbg_host_alloc(nbytes, C.byref(self.ptr)))

    def __del__(self):
        try:
            if self.ptr:
                lib().mbg_host_free(self.ptr)
                self.ptr = None
        except Exception:
            pass


def pinned_empty(n: int, dtype=np.float64) -> np.ndarray:
    """A numpy array in page-locked host memory (DMA'd directly by solve_host)."""
    dt = np.dtype(dtype)
    blk = _PinnedBlock(max(1, n * dt.itemsize))
    buf = (C.c_char * max(1, n * dt.itemsize)).from_address(blk.ptr.value)
    buf._owner = blk   # the array's base (buf) keeps the pinned block alive
    return np.frombuffer(buf, dtype=dt, count=n)

