"""Host-side logic of the product library (no GPU): generators, traffic
analyzer / schedules (Table 2), byte model, CSR validation, exact-dot limb
format and the halo plan."""
import json
from fractions import Fraction
from pathlib import Path

import numpy as np
import pytest

import oracle_ctypes as O
import paper_1907_12874_b200 as P

GOLD = json.loads((Path(__file__).parent / "golden" / "reference_fixtures.json").read_text())


def bits(a):
    return np.ascontiguousarray(a, dtype=np.float64).view(np.int64)


@pytest.mark.parametrize("kind,dims,seed", [("poisson7", (32, 32, 32), 0), ("convdiff7", (17, 9, 5), 1),
                                            ("stencil27", (12, 7, 9), 2), ("stencil27", (1, 1, 1), 2),
                                            ("convdiff7", (1, 5, 1), 3)])
def test_product_generators_equal_oracle(kind, dims, seed):
    a = P.gen_stencil(kind, *dims, seed=seed)
    o = O.gen_stencil(kind, *dims, seed=seed)
    assert np.array_equal(a.row_offsets, o.off) and np.array_equal(a.col_indices, o.col)
    assert np.array_equal(bits(a.values), bits(o.val))
    a.validate()


def test_product_banded_equals_oracle():
    a = P.gen_banded(150_000, 65536, 16, 32, 4)
    o = O.gen_banded(150_000, 65536, 16, 32, 4)
    assert np.array_equal(a.row_offsets, o.off) and np.array_equal(a.col_indices, o.col)
    assert np.array_equal(bits(a.values), bits(o.val))
    counts = np.diff(a.row_offsets)
    assert counts.min() >= 16 and counts.max() <= 32
    a.validate()
    # diagonal dominance 1.1 * sum |offdiag|
    i = 777
    cols = a.col_indices[a.row_offsets[i]:a.row_offsets[i + 1]]
    vals = a.values[a.row_offsets[i]:a.row_offsets[i + 1]]
    assert np.isclose(vals[cols == i][0], 1.1 * np.abs(vals[cols != i]).sum())
    # tiny n: band clipped, counts capped by available columns
    t = P.gen_banded(5, 65536, 16, 32, 4)
    assert np.all(np.diff(t.row_offsets) == 5)


def test_product_rhs_equals_oracle():
    assert np.array_equal(bits(P.gen_rhs(1000, 8, 3)), bits(O.rhs(1000, 8, 3)))
    b = P.gen_rhs(100_000, 2, 1)
    assert -1.0 <= b.min() < -0.99 and 0.99 < b.max() < 1.0


TABLE2 = {  # PAPER.md:343-363 (merged / basic) + 2 identity-M^-1 copies for Reordered
    ("bicgstab", "merged"): (14, 4), ("bicgstab", "basic"): (18, 4),
    ("rbicgstab", "merged"): (15 + 2, 6 + 2), ("rbicgstab", "basic"): (22 + 2, 6 + 2),
    ("pipebicgstab", "merged"): (18, 8), ("pipebicgstab", "basic"): (34, 9),
}


@pytest.mark.parametrize("key", list(TABLE2))
def test_method_schedule_table2(key):
    s = P.method_schedule(*key)
    assert (s["reads"], s["writes"]) == TABLE2[key]
    assert s["spmvs"] == 2


def test_method_schedule_reductions():
    # Eq. (14) / (16) / (18): message layout of the reductions
    assert P.method_schedule("bicgstab")["reductions"] == [1, 3, 1]
    assert P.method_schedule("rbicgstab")["reductions"] == [1, 4]
    assert P.method_schedule("pipebicgstab")["reductions"] == [3, 4]
    assert P.method_schedule("bicgstab", "basic")["reductions"] == [1] * 5


EQ14_19 = {  # merged vector transfers of Eqs. (14)-(19), preconditioner apart
    "bicgstab": (18, 0, [1, 3, 1]), "ibicgstab": (20, 0, [7]), "pipebicgstab": (26, 0, [3, 4]),
    "pbicgstab": (19, 2, [1, 3, 1]), "rbicgstab": (21, 2, [1, 4]), "ppipebicgstab": (34, 2, [3, 4]),
}


@pytest.mark.parametrize("method", list(EQ14_19))
def test_method_schedule_pc_eq14_19(method):
    s = P.method_schedule_pc(method)
    assert (s["vec"], s["precond"], s["reductions"]) == EQ14_19[method]
    assert s["spmvs"] == 2


def test_method_schedule_pc_variants():
    # basic: every dot its own reduction; split_basic peels the 4-vector updates of Alg. 7
    assert P.method_schedule_pc("ibicgstab", "basic")["reductions"] == [1] * 7
    pp = P.method_schedule_pc("ppipebicgstab", "basic")
    assert pp["reductions"] == [1] * 7 and pp["vec"] > 34
    # fused + identity: the M^-1 copies are elided; a synthetic preconditioner is not
    assert P.method_schedule_pc("pbicgstab", "fused")["precond"] == 0
    assert P.method_schedule_pc("pbicgstab", "fused", 4)["precond"] == 2
    # legacy totals fold one read + one write per identity application in
    assert P.method_schedule("pbicgstab")["reads"] == 15 + 2
    assert P.method_schedule("ppipebicgstab")["writes"] == 11 + 2
    with pytest.raises(ValueError):
        P.method_schedule_pc("bicgstab", "merged", 2)
    with pytest.raises(ValueError):
        P.method_schedule_pc("pbicgstab", "merged", 3)


# merged lines as (kind, ...) tuples with symbolic vector ids
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


def to_group(g):
    one = np.ones(1)
    out = []
    for st in g:
        if st[0] == "u":
            out.append(P.UpdateStatement(st[1], [(one, v) for v in st[2]]))
        else:
            out.append(P.DotStatement(st[1], st[2], st[3]))
    return out


@pytest.mark.parametrize("method", list(GROUPS))
def test_analyzer_matches_reference_analyzer(method):
    """Per merged line, analyze_traffic / split_basic equal the reference's
    (statement.cpp:25-85, golden fixture generated from the reference)."""
    for g, want in zip(GROUPS[method], GOLD["traffic"][method]):
        grp = to_group(g)
        assert list(P.analyze_traffic(grp)) == want["merged"]
        r, w, n = P.split_basic_traffic(grp, 100)
        assert [r, w] == want["basic"] and n == want["pieces"]


def test_analyzer_spec_examples():
    one = np.ones(2)
    # y = a x + b y -> (2, 1)
    assert P.analyze_traffic([P.UpdateStatement(1, [(one, 0), (one, 1)])]) == (2, 1)
    # w = y - omega (t - alpha v) splits through one temporary: 2x(2,1)
    r, w, n = P.split_basic_traffic([P.UpdateStatement(0, [(one, 1), (one, 2), (one, 3)])], 100)
    assert (r, w, n) == (4, 2, 2)
    # dot (v, v) counts v once; empty group
    assert P.analyze_traffic([P.DotStatement(3, 3, 0)]) == (1, 0)
    assert P.analyze_traffic([]) == (0, 0)
    with pytest.raises(ValueError, match="dangling"):
        P.analyze_traffic([P.DotStatement(-1, 0, 0)])


def test_byte_models():
    assert P.spmv_traffic_bytes(8_000_000, 56_000_000, 1) == GOLD["spmv_traffic_bytes_8e6_m1_C7"]
    if O.ref_available():
        for n, nnz, m in [(1000, 6000, 1), (8000, 55000, 4), (33, 200, 16)]:
            assert P.spmv_traffic_bytes(n, nnz, m) == O.ref().ref_spmv_traffic_bytes(n, nnz, m)
    n, nnz, m = 2_097_152, 14_581_760, 8
    assert P.spmv_compulsory_bytes(n, nnz, m) == 16 * m * n + 12 * nnz + 4 * (n + 1)


def test_csr_validate_messages_match_reference():
    good = O.gen_stencil("poisson7", 3, 3, 3)
    P.CsrMatrix(good.n, good.off, good.col, good.val).validate()
    bad_cols = good.col.copy()
    bad_cols[5], bad_cols[6] = bad_cols[6], bad_cols[5]
    cases = [
        (P.CsrMatrix(good.n, good.off, bad_cols, good.val), "not strictly increasing in row"),
        (P.CsrMatrix(good.n, good.off, np.where(good.col == 4, 99, good.col), good.val), "out of range"),
        (P.CsrMatrix(good.n, np.concatenate([[1], good.off[1:]]), good.col, good.val), "row_offsets\\[0\\]"),
    ]
    for a, msg in cases:
        with pytest.raises(ValueError, match=msg) as ei:
            a.validate()
        if O.ref_available():
            lib = O.ref()
            assert lib.ref_validate(a.n_rows, a.row_offsets, a.col_indices, a.values) == 1
            assert lib.ref_last_error().decode() == str(ei.value)


# --------------------------------------------------------------------------
# exact-dot limb format (host hooks share exact.cuh with the device)
# --------------------------------------------------------------------------
def test_exact_limbs_vs_fraction_and_partition_independent():
    rng = np.random.default_rng(11)
    n, m = 6000, 3
    a = rng.standard_normal(n * m) * np.exp2(rng.integers(-300, 300, n * m))
    b = rng.standard_normal(n * m)
    whole = P.exact_round(P.exact_accumulate(a, b, m), m)
    for c in range(m):
        want = float(sum((Fraction(float(p)) for p in a[c::m] * b[c::m]), Fraction(0)))
        assert whole[c] == want
    # any split of the rows, limbs summed as int64: identical result
    cuts = np.sort(rng.choice(np.arange(1, n), 5, replace=False))
    parts = np.split(np.arange(n), cuts)
    acc = np.zeros(m * P.exact_slot_words(), np.int64)
    for rows in parts:
        idx = (rows[:, None] * m + np.arange(m)).reshape(-1)
        acc += P.exact_accumulate(a[idx], b[idx], m)
    assert np.array_equal(bits(P.exact_round(acc, m)), bits(whole))
    assert np.array_equal(bits(whole), bits(O.dot_exact(a, b, m)))


def test_exact_round_edge_cases():
    w = P.exact_slot_words()
    cases = [np.array([2.0 ** 53, 1.0]), np.array([2.0 ** 53, 1.0, 2.0 ** -60]), np.array([5e-324, 5e-324]),
             np.array([1e308, 1e308, -1e308]), np.array([1.7e308, 1.7e308]), np.array([-3.0, 3.0]),
             np.array([-1e-300, 1e-310]), np.array([np.inf, 2.0]), np.array([np.inf, -np.inf])]
    for v in cases:
        got = P.exact_round(P.exact_accumulate(v, np.ones_like(v), 1), 1)[0]
        want = O.sum_exact(v)
        assert (np.isnan(got) and np.isnan(want)) or bits(got) == bits(want), (v, got, want)
    assert w == 72


# --------------------------------------------------------------------------
# halo plan (single process view of every part)
# --------------------------------------------------------------------------
@pytest.mark.parametrize("nparts", [1, 2, 3, 5])
def test_halo_plan_consistent(nparts):
    a = P.gen_banded(3000, 400, 4, 12, 9)
    n = a.n_rows
    bounds = [n * p // nparts for p in range(nparts + 1)]
    plans = [P.halo_plan(a, bounds, p) for p in range(nparts)]
    for p, pl in enumerate(plans):
        r0, r1 = bounds[p], bounds[p + 1]
        assert pl["n_own"] == r1 - r0
        # local column -> global column reproduces the CSR, order preserved
        glob = np.concatenate([np.arange(r0, r1), pl["halo_global"]])
        sl = slice(a.row_offsets[r0], a.row_offsets[r1])
        assert np.array_equal(glob[pl["col"]], a.col_indices[sl])
        assert np.array_equal(bits(pl["val"]), bits(a.values[sl]))
        # my receive window from q == q's send list to me
        for peer in pl["peers"]:
            q = peer["part"]
            mine = pl["halo_global"][peer["recv_offset"]:peer["recv_offset"] + peer["recv_count"]]
            theirs = [x for x in plans[q]["peers"] if x["part"] == p]
            sent = theirs[0]["send_rows"] + bounds[q] if theirs else np.zeros(0, np.int64)
            assert np.array_equal(mine, sent)


def test_method_schedule_fused_reordered():
    # fused Reordered (identity M^-1 elided): the delta dot in the SpMM epilogue
    # reads one aux vector; rt stays in registers and r = rt - omega t rides in
    # the x / z / vh pass: 17 group transfers + 1 aux = 18 (merged listing: 21 + 4)
    s = P.method_schedule_pc("rbicgstab", "fused")
    assert s["vec"] == 18 and s["precond"] == 0 and s["reductions"] == [1, 4]


def test_method_schedule_fused_pipelined():
    # fused Pipelined: lines 7 + 12 in one pass and q, y in registers only
    # (formed for the line-4 dots, recomputed in the line-7/12 pass): 22 (merged 26)
    s = P.method_schedule_pc("pipebicgstab", "fused")
    assert s["vec"] == 22 and s["reductions"] == [3, 4]


def test_sorted_twin_plan_properties():
    """Host logic of the CSR SpMM's length-sorted twin: a permutation of the
    rows (long rows last, one slot each), descending lengths inside each
    window, stable (ties keep the row order), groups of 8 slots with the
    batches of their longest row, tiles of whole groups within a stage."""
    rng = np.random.default_rng(5)
    n, window = 10_001, 512
    lens = rng.integers(0, 41, n)
    lens[[17, 4000, 9000]] = [240, 241, 3000]   # the longest row of the twin, two beyond it
    off = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    plan = P.sorted_twin_plan(off, window)
    rowid, tiles, goff = plan["rowid"], plan["tiles"], plan["group_off"]
    nreg = n - 2
    nslots = (nreg + 7) // 8 * 8
    assert rowid.size == nslots + 2
    assert list(rowid[nslots:]) == [4000, 9000]
    assert np.all(rowid[nreg:nslots] == -1)
    assert np.array_equal(np.sort(rowid[rowid >= 0]), np.arange(n))
    reg = np.array([r for r in range(n) if r not in (4000, 9000)])
    for w0 in range(0, nreg, window):
        seg = rowid[w0:min(nreg, w0 + window)]
        assert set(seg.tolist()) == set(reg[w0:w0 + window].tolist())
        ls = lens[seg]
        assert np.all(np.diff(ls) <= 0)
        for v in np.unique(ls):                  # stable: equal lengths keep ascending rows
            assert np.all(np.diff(seg[ls == v]) > 0)
    G = nslots // 8
    nb = np.array([max([(lens[r] + 3) // 4 for r in rowid[8 * g:8 * g + 8] if r >= 0], default=0) for g in range(G)])
    assert np.array_equal(goff[:G + 1], np.concatenate([[0], np.cumsum(nb)]))
    reg_t, long_t = tiles[tiles[:, 2] >= 0], tiles[tiles[:, 2] < 0]
    assert reg_t[0, 0] == 0 and reg_t[-1, 1] == nslots
    assert np.array_equal(reg_t[1:, 0], reg_t[:-1, 1]) and np.all(reg_t[:, 0] % 8 == 0)
    assert np.array_equal(reg_t[:, 2], goff[reg_t[:, 0] // 8]) and np.array_equal(reg_t[:, 3], goff[reg_t[:, 1] // 8])
    assert np.all(reg_t[:, 3] - reg_t[:, 2] <= 60) and np.all(reg_t[:, 1] - reg_t[:, 0] <= 192)
    assert np.array_equal(long_t[:, 0], [nslots, nslots + 1]) and np.all(long_t[:, 3] == -1)
    assert 0.5 < plan["lane_efficiency"] < 0.9
    # uniform rows: nothing to gain
    assert P.sorted_twin_plan(np.arange(0, 7 * 1000 + 1, 7), 4096)["lane_efficiency"] == 1.0


def test_infer_grid_host_logic(monkeypatch):
    """Grid detection's host half (api.cu infer_grid): the longest row's column
    offsets give nx, ny, nz for lexicographic 7- / 27-point operators; other
    matrices give none."""
    monkeypatch.setenv("MBG_AUTO_GRID", "1")
    for kind, dims in (("poisson7", (16, 16, 16)), ("convdiff7", (24, 20, 9)), ("convdiff7", (3, 5, 4)),
                       ("stencil27", (13, 11, 10)), ("stencil27", (3, 3, 3)), ("stencil27", (40, 3, 7))):
        a = O.gen_stencil(kind, *dims, seed=2)
        assert P.infer_grid(P.CsrMatrix(a.n, a.off, a.col, a.val)) == dims, (kind, dims)
    band = O.gen_banded(5000, 300, 16, 32, 4)
    assert P.infer_grid(P.CsrMatrix(band.n, band.off, band.col, band.val)) == (0, 0, 0)
    tiny = O.gen_stencil("poisson7", 2, 2, 2)            # no interior point
    assert P.infer_grid(P.CsrMatrix(tiny.n, tiny.off, tiny.col, tiny.val)) == (0, 0, 0)
    # a 2-D five-point operator (one plane) is not a 3-D grid operator
    flat = O.gen_stencil("poisson7", 12, 12, 1)
    assert P.infer_grid(P.CsrMatrix(flat.n, flat.off, flat.col, flat.val)) == (0, 0, 0)
    monkeypatch.setenv("MBG_AUTO_GRID", "0")
    a = O.gen_stencil("poisson7", 8, 8, 8)
    assert P.infer_grid(P.CsrMatrix(a.n, a.off, a.col, a.val)) == (0, 0, 0)
