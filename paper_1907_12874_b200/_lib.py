"""ctypes binding of the C ABI (include/mbstab_b200.h).

The shared library is built in-tree (``paper_1907_12874_b200/libmbstab_b200.so``,
see csrc/Makefile).  There is no fallback: if it is missing or fails to load,
every entry point raises.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

HERE = Path(__file__).resolve().parent
# MBG_CHECKED=1: the guard-zone build (csrc/Makefile `checked`), for the
# out-of-bounds tests that stand in for compute-sanitizer on this pool
LIB_PATH = HERE / ("libmbstab_b200_checked.so" if os.environ.get("MBG_CHECKED") == "1" else "libmbstab_b200.so")
if os.environ.get("MBG_LIB"):   # A/B measurements: another build of the same library (tools/ncu_ab.sh)
    LIB_PATH = Path(os.environ["MBG_LIB"]).resolve()

MBG_OK, MBG_ERR_INVALID, MBG_ERR_RUNTIME, MBG_ERR_BREAKDOWN = 0, 1, 2, 3
MBG_MAX_TERMS = 8


class MbgStatement(C.Structure):
    _fields_ = [
        ("kind", C.c_int),
        ("out", C.c_int),
        ("nterms", C.c_int),
        ("term_vec", C.c_int * MBG_MAX_TERMS),
        ("term_coeff", C.c_void_p * MBG_MAX_TERMS),
        ("left", C.c_int),
        ("right", C.c_int),
        ("slot", C.c_int),
    ]


class MbgReport(C.Structure):
    _fields_ = [
        ("iterations", C.c_int),
        ("converged", C.c_int),
        ("breakdown", C.c_int),
        ("breakdown_iter", C.c_int),
        ("breakdown_col", C.c_int),
        ("vector_reads", C.c_int64),
        ("vector_writes", C.c_int64),
        ("spmv_bytes", C.c_double),
        ("compulsory_bytes", C.c_double),
        ("reductions", C.c_int64),
        ("gpu_launches", C.c_int64),
        ("loop_ms", C.c_double),
    ]


class BreakdownError(RuntimeError):
    """Solver breakdown: a denominator vanished."""


_lib = None


def build() -> None:
    """Compile the CUDA library in-tree (nvcc, sm_100a)."""
    import subprocess
    subprocess.run(["make", "-s", "-j", str(os.cpu_count() or 4), "-C", str(HERE / "csrc")], check=True)


def lib() -> C.CDLL:
    global _lib
    if _lib is not None:
        return _lib
    if not LIB_PATH.exists():
        raise RuntimeError(
            f"{LIB_PATH} is missing: build it with `make -C {HERE / 'csrc'}` "
            "(the B200 path has no CPU fallback)")
    L = C.CDLL(str(LIB_PATH))
    vp, i64, i32, dbl, ip = C.c_void_p, C.c_int64, C.c_int, C.c_double, C.POINTER(C.c_int)
    pp = C.POINTER(C.c_void_p)
    sig = {
        "mbg_last_error": (C.c_char_p, []),
        "mbg_version": (C.c_char_p, []),
        "mbg_ctx_create": (i32, [i32, pp]),
        "mbg_ctx_destroy": (i32, [vp]),
        "mbg_ctx_synchronize": (i32, [vp]),
        "mbg_comm_unique_id": (i32, [C.c_char_p]),
        "mbg_ctx_init_comm": (i32, [vp, i32, i32, C.c_char_p]),
        "mbg_local_group_create": (i32, [vp, i32]),
        "mbg_csr_validate": (i32, [i64, vp, vp, i64]),
        "mbg_csr_upload": (i32, [vp, i64, vp, vp, vp, pp]),
        "mbg_csr_upload_partitioned": (i32, [vp, i64, vp, vp, vp, i32, vp, i32, pp]),
        "mbg_halo_plan": (i32, [i64, vp, vp, vp, i32, vp, i32, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp,
                                vp, vp]),
        "mbg_transpose_halo_plan": (i32, [i64, vp, vp, vp, i32, vp, i32, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp,
                                vp, vp]),
        "mbg_csr_free": (i32, [vp]),
        "mbg_csr_rows": (i64, [vp]),
        "mbg_csr_nnz": (i64, [vp]),
        "mbg_csr_stage_info": (i32, [vp, vp, vp]),
        "mbg_csr_sort_info": (i32, [vp, vp, vp]),
        "mbg_sorted_twin_plan": (i32, [i64, vp, i32, vp, vp, vp, vp, vp, vp]),
        "mbg_csr_upload_any_order": (i32, [vp, i64, vp, vp, vp, pp]),
        "mbg_csr_set_grid": (i32, [vp, vp, i32, i32, i32]),
        "mbg_csr_clear_grid": (i32, [vp]),
        "mbg_infer_grid": (i32, [i64, vp, vp, vp, vp, vp]),
        "mbg_spmv_transpose": (i32, [vp, vp, vp, vp]),
        "mbg_true_residual": (i32, [vp, vp, vp, vp, vp]),
        "mbg_csr_reordered": (i32, [vp]),
        "mbg_csr_stencil_kind": (i32, [vp]),
        "mbg_ctx_set_small_path": (i32, [vp, i32]),
        "mbg_ctx_reserve_sms": (i32, [vp, i32]),
        "mbg_debug_guard_check": (i32, [C.POINTER(C.c_int64)]),
        "mbg_debug_write_past_end": (i32, [vp]),
        "mbg_mv_alloc": (i32, [vp, i64, i32, pp]),
        "mbg_mv_free": (i32, [vp]),
        "mbg_mv_upload": (i32, [vp, vp]),
        "mbg_mv_download": (i32, [vp, vp]),
        "mbg_mv_fill": (i32, [vp, dbl]),
        "mbg_mv_device_ptr": (vp, [vp]),
        "mbg_spmv": (i32, [vp, vp, vp, vp]),
        "mbg_spmv_traffic_bytes": (dbl, [i64, i64, i32]),
        "mbg_spmv_compulsory_bytes": (dbl, [i64, i64, i32]),
        "mbg_analyze_traffic": (i32, [vp, i32, ip, ip]),
        "mbg_split_basic_traffic": (i32, [vp, i32, i32, ip, ip, ip]),
        "mbg_execute_group": (i32, [vp, vp, i32, vp, i32, vp, i32]),
        "mbg_solve": (i32, [vp, vp, vp, vp, i32, i32, dbl, i32, i32, vp, C.POINTER(MbgReport)]),
        "mbg_solve_pc": (i32, [vp, vp, vp, vp, i32, i32, i32, dbl, i32, i32, vp, C.POINTER(MbgReport)]),
        "mbg_solve_host": (i32, [vp, vp, i32, vp, vp, i32, i32, dbl, i32, i32, vp, C.POINTER(MbgReport)]),
        "mbg_solve_profile": (i32, [vp, vp, vp, vp, i32, i32, dbl, i32, i32, C.c_char_p, i32,
                                    C.POINTER(MbgReport)]),
        "mbg_method_schedule": (i32, [i32, i32, ip, ip, ip, ip, ip]),
        "mbg_method_schedule_pc": (i32, [i32, i32, i32, ip, ip, ip, ip, ip, ip]),
        "mbg_gen_stencil": (i32, [i32, i32, i32, i32, C.c_uint64, C.POINTER(C.c_int64), vp, vp, vp]),
        "mbg_gen_banded": (i32, [i64, i64, i32, i32, C.c_uint64, C.POINTER(C.c_int64), vp, vp, vp]),
        "mbg_gen_rhs": (i32, [i64, i32, C.c_uint64, vp]),
        "mbg_mm_read": (i32, [C.c_char_p, C.POINTER(C.c_void_p), C.POINTER(C.c_int64), C.POINTER(C.c_int64)]),
        "mbg_mm_copy": (i32, [vp, vp, vp, vp]),
        "mbg_mm_free": (None, [vp]),
        "mbg_mm_write": (i32, [C.c_char_p, i64, vp, vp, vp]),
        "mbg_fusion_bench": (i32, [vp, i64, i32, vp, vp, C.POINTER(C.c_int)]),
        "mbg_host_alloc": (i32, [C.c_size_t, C.POINTER(C.c_void_p)]),
        "mbg_host_free": (i32, [vp]),
        "mbg_exact_slot_words": (i32, []),
        "mbg_exact_accumulate_host": (i32, [i64, i32, vp, vp, vp]),
        "mbg_exact_round_host": (i32, [vp, i32, vp]),
        "mbg_ctx_launches": (i64, [vp]),
    }
    for name, (res, args) in sig.items():
        if os.environ.get("MBG_LIB") and not hasattr(L, name):
            continue   # an older build under A/B measurement: entry points added since are absent
        f = getattr(L, name)
        f.restype = res
        f.argtypes = args
    _lib = L
    return L


def check(rc: int) -> None:
    if rc == MBG_OK:
        return
    msg = lib().mbg_last_error().decode()
    if rc == MBG_ERR_INVALID:
        raise ValueError(msg)
    if rc == MBG_ERR_BREAKDOWN:
        raise BreakdownError(msg)
    raise RuntimeError(msg)
