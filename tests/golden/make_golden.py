"""Generate tests/golden/reference_fixtures.json from the REFERENCE's own code.

Runs in the build container only (needs oracle/_ref/libmbstab_ref.so, compiled
from /root/reference/proj sources by oracle/Makefile).  The committed JSON lets
the CPU suite pin the oracle against the reference where /root/reference is
absent (GPU box).  Fixtures:
  * gen_poisson_7pt outputs (generators.cpp:37-67) -- sha256 of the arrays;
  * spmv outputs (spmv.cpp:27-74) on fixed inputs for several m -- sha256;
  * execute_group outputs (execute.cpp:123-172) for the Alg. 2 x/r/rho group;
  * analyze_traffic / split_basic counts (statement.cpp:25-85) for every merged
    line of Alg. 2, 4 and 6 (these sum to Table 2);
  * spmv_traffic_bytes (spmv.cpp:10-16) on the SPEC.md:74 example.

usage: python tests/golden/make_golden.py
"""
import ctypes as C
import hashlib
import json
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parent))
sys.path.insert(0, str(HERE.parent.parent))
import oracle_ctypes as O  # noqa: E402
from paper_1907_12874_b200._lib import MbgStatement  # noqa: E402  (plain C struct layout)


def sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def x_input(n, m):
    i = np.arange(n * m, dtype=np.float64)
    return np.sin(0.37 * i + 0.1) * (1.0 + (i % 7))


def stmt_array(group):
    arr = (MbgStatement * len(group))()
    keep = []
    for k, st in enumerate(group):
        s = arr[k]
        if st[0] == "u":
            _, out, terms = st
            s.kind, s.out, s.nterms = 0, out, len(terms)
            for t, v in enumerate(terms):
                c = np.full(1, 0.5 + t)
                keep.append(c)
                s.term_vec[t] = v
                s.term_coeff[t] = c.ctypes.data
        else:
            _, l, r, slot = st
            s.kind, s.left, s.right, s.slot = 1, l, r, slot
    return arr, keep


# merged lines with symbolic ids
X, P_, R, R0, V, S, T, Z, VH, TH, RT, Q, W, Y = range(14)
GROUPS = {
    "bicgstab": [[("d", V, R0, 0)], [("u", S, [R, V])], [("d", T, S, 0), ("d", T, T, 1), ("d", S, S, 2)],
                 [("u", X, [X, P_, S]), ("u", R, [S, T]), ("d", R, R0, 0)], [("u", P_, [R, P_, V])]],
    "rbicgstab": [[("d", V, R0, 0)], [("u", TH, [Z, S])],
                  [("u", RT, [R, V]), ("d", T, RT, 0), ("d", T, T, 1), ("d", T, R0, 2), ("d", RT, RT, 3)],
                  [("u", R, [RT, T])], [("u", X, [X, VH, TH]), ("u", Z, [TH, Q]), ("u", VH, [Z, VH, S])]],
    "pipebicgstab": [[("u", P_, [R, P_, S]), ("u", S, [W, S, Z]), ("u", Z, [T, Z, V]), ("u", Q, [R, S]),
                      ("u", Y, [W, Z]), ("d", Q, Y, 0), ("d", Y, Y, 1), ("d", Q, Q, 2)],
                     [("u", X, [X, P_, Q]), ("u", R, [Q, Y])],
                     [("u", W, [Y, T, V]), ("d", R0, R, 0), ("d", R0, Z, 1), ("d", R0, W, 2), ("d", R0, S, 3)]],
}


def main():
    ref = O.ref()
    out = {"generator": "tests/golden/make_golden.py (reference compiled from /root/reference/proj)"}
    gens = {}
    for dims in [(1, 1, 1), (2, 2, 2), (3, 4, 5), (6, 5, 4)]:
        a = O.ref_gen_poisson_7pt(*dims)
        gens["x".join(map(str, dims))] = {"n": a.n, "nnz": a.nnz, "off": sha(a.off), "col": sha(a.col),
                                          "val": sha(a.val)}
    out["gen_poisson_7pt"] = gens
    a = O.ref_gen_poisson_7pt(6, 5, 4)
    sp = {}
    for m in (1, 3, 8):
        y = O.ref_spmv(a, x_input(a.n, m), m, threads=3)
        sp[str(m)] = sha(y)
    out["spmv_poisson7_6x5x4"] = sp
    out["spmv_traffic_bytes_8e6_m1_C7"] = ref.ref_spmv_traffic_bytes(8_000_000, 56_000_000, 1)

    # execute_group: Alg. 2 x/r/rho group on fixed vectors, m = 3, one thread
    n, m = 97, 3
    vecs = [x_input(n, m) * (k + 1) + k for k in range(6)]  # x p s t r0 r
    alpha = np.array([0.3, -1.25, 2.0])
    omega = np.array([-0.7, 0.125, 1.5])
    one = np.ones(m)
    grp = (MbgStatement * 3)()
    keep = [alpha, omega, one, -omega]
    g0, g1, g2 = grp[0], grp[1], grp[2]
    g0.kind, g0.out, g0.nterms = 0, 0, 3
    for t, (c, v) in enumerate([(one, 0), (alpha, 1), (omega, 2)]):
        g0.term_vec[t], g0.term_coeff[t] = v, c.ctypes.data
    g1.kind, g1.out, g1.nterms = 0, 5, 2
    for t, (c, v) in enumerate([(one, 2), (keep[3], 3)]):
        g1.term_vec[t], g1.term_coeff[t] = v, c.ctypes.data
    g2.kind, g2.left, g2.right, g2.slot = 1, 5, 4, 0
    ptrs = (C.c_void_p * 6)(*[v.ctypes.data for v in vecs])
    dots = np.zeros(m)
    ref.ref_run_group.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_int64, C.c_int, C.c_void_p, C.c_void_p,
                                  C.c_int, C.c_int]
    assert ref.ref_run_group(grp, 3, 6, n, m, ptrs, dots.ctypes.data, 1, 1) == 0
    out["execute_group_alg2_xr"] = {"n": n, "m": m, "x": sha(vecs[0]), "r": sha(vecs[5]),
                                    "rho": [float(d) for d in dots]}

    ref.ref_analyze_traffic.argtypes = [C.c_void_p, C.c_int, C.c_int, C.POINTER(C.c_int), C.POINTER(C.c_int)]
    ref.ref_split_basic_traffic.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_int, C.POINTER(C.c_int),
                                            C.POINTER(C.c_int), C.POINTER(C.c_int)]
    tr = {}
    for meth, groups in GROUPS.items():
        rows = []
        for g in groups:
            arr, keep = stmt_array(g)
            r, w, r2, w2, ng = C.c_int(), C.c_int(), C.c_int(), C.c_int(), C.c_int()
            assert ref.ref_analyze_traffic(arr, len(g), 1, C.byref(r), C.byref(w)) == 0
            assert ref.ref_split_basic_traffic(arr, len(g), 1, 100, C.byref(r2), C.byref(w2), C.byref(ng)) == 0
            rows.append({"merged": [r.value, w.value], "basic": [r2.value, w2.value], "pieces": ng.value})
        tr[meth] = rows
    out["traffic"] = tr
    (HERE / "reference_fixtures.json").write_text(json.dumps(out, indent=1) + "\n")
    print("wrote", HERE / "reference_fixtures.json")


if __name__ == "__main__":
    main()
