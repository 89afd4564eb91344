"""The paper's execution-time model (PAPER.md:541-785,
SPEC.md:280-392): known answers from SPEC.md, the Table 5 validation points,
the schedule bridge to the solver's own transfer counts, and the qualitative
structure of Figs. 5-8."""
import dataclasses

import pytest

import paper_1907_12874_b200 as P
from paper_1907_12874_b200 import perfmodel as M

L2 = M.LOMONOSOV2
SPEC = M.ProblemSpec(N=8e6, m=1, C=7)


def test_t_vec_and_sigma_mul():
    assert M.t_vec(L2, SPEC, 1) == pytest.approx(1.0667e-3, rel=1e-4)
    assert M.t_vec(L2, dataclasses.replace(SPEC, m=2), 1) == pytest.approx(2 * M.t_vec(L2, SPEC, 1))
    assert M.t_vec(L2, SPEC, 2) == pytest.approx(M.t_vec(L2, SPEC, 1) / 2)
    assert M.sigma_mul(M.ProblemSpec(N=1, m=1, C=0)) == 12
    assert M.sigma_mul(M.ProblemSpec(N=8e6, m=4, C=7)) == pytest.approx(2.752e9)
    assert M.t_mul(L2, SPEC, 1) == pytest.approx(0.02027, rel=1e-3)


def test_local_and_global_fits():
    assert M.t_local(L2, 0) == pytest.approx(2.4e-6)
    assert M.t_local(L2, 2048) == pytest.approx(7.33e-6, rel=2e-3)
    assert M.t_local(L2, 2049) == pytest.approx(7.30e-6, rel=2e-3)
    assert M.t_global(L2, 1, 8) == pytest.approx(6.13e-6, rel=2e-3)
    assert M.t_global(L2, 128, 24) == pytest.approx(4.9e-5, rel=2e-2)
    flat = dataclasses.replace(L2, global_fit=M.GlobalFit(5e-6, 0.0, 0.21, 0.54))
    assert M.t_global(flat, 77, 1000) == 5e-6


def test_overlap_rule():
    assert M.overlapped(10e-6, 4e-6, 1.0) == pytest.approx(14e-6)
    assert M.overlapped(10e-6, 4e-6, 0.0) == pytest.approx(10e-6)
    assert M.overlapped(10e-6, 4e-6, 0.5) == pytest.approx(12e-6)
    for g in (0.0, 0.3, 1.0):
        v = M.overlapped(3e-6, 5e-6, g)
        assert max(3e-6, 5e-6) <= v <= 8e-6 + 1e-18


def test_table5_validation_points():
    """PAPER Table 5 (Lomonosov-2, N=8e6, m=1): BiCGStab 0.057, PPipeBiCGStab 0.077."""
    assert 0.057 <= M.t_iteration(L2, SPEC, "bicgstab", 1) <= 0.060
    pp = dataclasses.replace(SPEC, precond_alpha=2)
    assert 0.077 <= M.t_iteration(L2, pp, "ppipebicgstab", 1) <= 0.082


@pytest.mark.parametrize("method", list(M.VEC))
def test_schedule_bridge(method):
    """The model's vector coefficients equal the solver's merged schedule."""
    s = P.method_schedule_pc(method, "merged")
    assert s["vec"] == M.VEC[method]
    assert s["precond"] == (2 if method in M.PRECONDITIONED else 0)


def test_preconditioner_consistency():
    with pytest.raises(ValueError):
        M.t_iteration(L2, SPEC, "pbicgstab", 1)
    with pytest.raises(ValueError):
        M.t_iteration(L2, dataclasses.replace(SPEC, precond_alpha=2), "bicgstab", 1)


def test_gamma_only_moves_reduction_terms():
    g1 = dataclasses.replace(L2, gamma=1.0)
    g0 = dataclasses.replace(L2, gamma=0.0)
    # one node: no reductions, gamma irrelevant
    assert M.t_iteration(g1, SPEC, "pipebicgstab", 1) == M.t_iteration(g0, SPEC, "pipebicgstab", 1)
    assert M.t_iteration(g1, SPEC, "pipebicgstab", 64) >= M.t_iteration(g0, SPEC, "pipebicgstab", 64)


def test_monotonicity():
    for mth in M.VEC:
        spec = dataclasses.replace(SPEC, precond_alpha=2 if mth in M.PRECONDITIONED else 0)
        for p in (1, 8, 64):
            t = M.t_iteration(L2, spec, mth, p)
            assert M.t_iteration(dataclasses.replace(L2, b=2 * L2.b), spec, mth, p) <= t
            assert M.t_iteration(L2, dataclasses.replace(spec, m=2), mth, p) >= t
            if mth in M.PRECONDITIONED:
                assert M.t_iteration(L2, dataclasses.replace(spec, precond_alpha=6), mth, p) >= t


def spec_of(mth, base=SPEC):
    return dataclasses.replace(base, precond_alpha=2 if mth in M.PRECONDITIONED else 0)


def test_relative_performance_table():
    rel = M.relative_performance(dataclasses.replace(M.LOMONOSOV, gamma=1.0), spec_of,
                                 ["bicgstab", "ibicgstab", "pipebicgstab"], range(1, 129))
    for p, r in rel.items():
        assert max(r.values()) == pytest.approx(1.0) and all(0 < v <= 1 for v in r.values())
    # p = 1: the fewest transfers win (classical)
    assert max(rel[1], key=rel[1].get) == "bicgstab"
    # gamma = 1: a crossover to IBiCGStab (one reduction) exists in [2, 128]
    assert any(max(rel[p], key=rel[p].get) == "ibicgstab" for p in range(2, 129))


def test_pipelined_wins_an_interval_with_gamma0():
    rel = M.relative_performance(dataclasses.replace(M.LOMONOSOV, gamma=0.0), spec_of,
                                 ["bicgstab", "ibicgstab", "pipebicgstab"], range(1, 513))
    assert any(max(r, key=r.get) == "pipebicgstab" for r in rel.values())


def test_breakeven_and_speedups():
    assert M.breakeven_elements(20e-6, 1e11) == pytest.approx(2.5e5)
    assert M.breakeven_elements(0.0, 1e11) == 0.0
    times = {p: M.t_iteration(L2, SPEC, "bicgstab", p) for p in (1, 2, 4)}
    s = M.speedup(times)
    assert s[1] == 1.0 and s[4] > s[2] > 1.0
    rs = M.relative_speedup({"bicgstab": times, "ibicgstab": {p: M.t_iteration(L2, SPEC, "ibicgstab", p)
                                                              for p in (1, 2, 4)}})
    assert rs["bicgstab"][1] == 1.0


def test_scan_rows():
    rows = M.scan(M.LOMONOSOV, SPEC, ["bicgstab", "rbicgstab"], [1, 4], [0.0, 1.0], [2], [1, 4])
    assert len(rows) == 2 * 2 * 2 * 1 * 2 * 2   # methods x p x gamma x bw modes x alpha x m
    one = M.scan(M.LOMONOSOV, SPEC, ["bicgstab"], [1], [1.0], [2], [1])
    assert all(r["R"] == 1.0 for r in one)
    with pytest.raises(ValueError):
        M.scan(M.LOMONOSOV, SPEC, [], [1], [1.0], [2], [1])


def test_fit_bandwidth():
    b = M.fit_bandwidth([1e9, 2e9, 3e9], [1e-3, 2e-3, 3e-3])
    assert b == pytest.approx(1e12)
