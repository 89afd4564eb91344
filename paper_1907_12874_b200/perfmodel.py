"""Data-transfer execution-time model of the paper.

Restates PAPER.md:541-785 / SPEC.md:280-392 as pure functions: T = Sigma / B
with B = b*p (Eq. (2)), the SpMV bytes of Eq. (3), T_vec of Eq. (6), the local
exchange fit T_L(l) (Eqs. (8)-(9)), the global reduction fit
T_G(p, l) = C0 + C1 l^n0 p^n1 (Eqs. (11)-(12)), the overlap rule
T = max(T_calc + gamma*T_G, T_G) (Eq. (13)) and the six per-iteration
estimators (Eqs. (14)-(19)).  The vector-transfer coefficients come from the
solver's own schedule (mbg_method_schedule_pc), so the model and the
instrumented GPU solver count the same transfers.

Presets: the paper's Lomonosov / Lomonosov-2 fits, and a B200 node whose
bandwidth is the measured HBM copy rate (MEASURED_PEAKS.json).  The B200
reduction fit is NOT measured here (one GPU in this environment): it is an
assumption stated in the preset (`measured=False`).
"""
from __future__ import annotations

import dataclasses
import math
from typing import Iterable, Sequence


@dataclasses.dataclass(frozen=True)
class LocalFit:           # Eq. (8)-(9): two branches split at `knee` bytes
    c0_small: float = 2.4e-6
    c1_small: float = 6.9e-8
    n0_small: float = 0.56
    c0_large: float = 3.2e-6
    c1_large: float = 2e-9
    knee: float = 2048.0


@dataclasses.dataclass(frozen=True)
class GlobalFit:          # Eq. (11)-(12)
    c0: float = 3.5e-6
    c1: float = 1.7e-6
    n0: float = 0.21
    n1: float = 0.54


@dataclasses.dataclass(frozen=True)
class MachineModel:
    name: str
    b: float                      # node memory bandwidth, bytes/s
    llc_b: float = 0.0            # last-level cache bandwidth, bytes/s (Table 6)
    local_fit: LocalFit = LocalFit()
    global_fit: GlobalFit = GlobalFit()
    gamma: float = 1.0            # overlapping overhead, Eq. (10)
    measured: bool = False        # were the fits measured on this machine?

    def __post_init__(self):
        if not (0.0 <= self.gamma <= 1.0):
            raise ValueError("gamma must lie in [0, 1]")
        if self.b <= 0:
            raise ValueError("bandwidth must be positive")


@dataclasses.dataclass(frozen=True)
class ProblemSpec:
    N: float                      # matrix rows (per job)
    m: int = 1                    # right-hand sides
    C: float = 7.0                # average nonzeros per row
    halo_bytes: float = 0.0       # average neighbour message l (p-independent, Sec. 3.1.3)
    precond_alpha: int = 0        # transfers per M^-1 application (0 = none)


LOMONOSOV = MachineModel("Lomonosov", b=16e9, llc_b=46e9)
LOMONOSOV_EFFECTIVE = MachineModel("Lomonosov (effective b, SPEC.md open question)", b=34e9, llc_b=46e9)
LOMONOSOV2 = MachineModel("Lomonosov-2", b=60e9)


def b200_node(hbm_gbs: float, gamma: float = 0.0) -> MachineModel:
    """One B200 per 'node'.  b = measured HBM copy bandwidth.  The reduction
    fit is an assumption (NCCL small-message allreduce over NVLink 5: ~10 us
    latency, weak growth with p) -- not measured in this one-GPU environment."""
    return MachineModel("B200 (b measured; T_G, T_L assumed)", b=hbm_gbs * 1e9,
                        local_fit=LocalFit(8e-6, 1e-9, 1.0, 8e-6, 1.0 / 450e9, 0.0),
                        global_fit=GlobalFit(10e-6, 0.5e-6, 0.21, 0.5), gamma=gamma, measured=False)


# ---- Eqs. (3)-(6) -------------------------------------------------------------
def sigma_mul(spec: ProblemSpec) -> float:
    """Eq. (3): SpMV bytes N(8m(C+1) + 4(3C+1))."""
    return spec.N * (8.0 * spec.m * (spec.C + 1.0) + 4.0 * (3.0 * spec.C + 1.0))


def sigma_mul_compulsory(spec: ProblemSpec) -> float:
    """x read once (the GPU roofline model): N(16m + 12C + 4)."""
    return spec.N * (16.0 * spec.m + 12.0 * spec.C + 4.0)


def t_vec(machine: MachineModel, spec: ProblemSpec, p: int) -> float:
    """Eq. (6): one vector transfer, 8Nm / (b p)."""
    _check_p(p)
    return 8.0 * spec.N * spec.m / (machine.b * p)


def t_mul(machine: MachineModel, spec: ProblemSpec, p: int, compulsory: bool = False) -> float:
    _check_p(p)
    return (sigma_mul_compulsory(spec) if compulsory else sigma_mul(spec)) / (machine.b * p)


def t_local(machine: MachineModel, l: float) -> float:
    """Eqs. (8)-(9): two-branch local exchange fit."""
    f = machine.local_fit
    if l <= f.knee:
        return f.c0_small + f.c1_small * l ** f.n0_small
    return f.c0_large + f.c1_large * l


def t_global(machine: MachineModel, p: int, l: float) -> float:
    """Eqs. (11)-(12): blocking allreduce of l = 8mk bytes over p nodes."""
    _check_p(p)
    g = machine.global_fit
    return g.c0 + g.c1 * l ** g.n0 * p ** g.n1


def t_spmv(machine: MachineModel, spec: ProblemSpec, p: int, compulsory: bool = False) -> float:
    """Eq. (15): max(T_mul, T_L(l)); no halo on one node."""
    tm = t_mul(machine, spec, p, compulsory)
    return tm if p == 1 or spec.halo_bytes <= 0 else max(tm, t_local(machine, spec.halo_bytes))


def overlapped(t_calc: float, t_g: float, gamma: float) -> float:
    """Eq. (13)."""
    return max(t_calc + gamma * t_g, t_g)


# ---- Eqs. (14)-(19) -------------------------------------------------------------
# merged vector transfers of each method (Eqs. (14)-(19)); equal to the solver's
# schedule (tests/test_perfmodel.py checks it against mbg_method_schedule_pc)
VEC = {"bicgstab": 18, "ibicgstab": 20, "pipebicgstab": 26, "pbicgstab": 19, "rbicgstab": 21,
       "ppipebicgstab": 34}
PRECONDITIONED = ("pbicgstab", "rbicgstab", "ppipebicgstab")


def t_iteration(machine: MachineModel, spec: ProblemSpec, method: str, p: int, compulsory: bool = False) -> float:
    pre = method in PRECONDITIONED
    if pre and spec.precond_alpha <= 0:
        raise ValueError(f"{method} needs a preconditioner (precond_alpha >= 2)")
    if not pre and spec.precond_alpha:
        raise ValueError(f"{method} takes no preconditioner")
    tv = t_vec(machine, spec, p)
    ts = t_spmv(machine, spec, p, compulsory)
    tp = spec.precond_alpha * tv
    g = machine.gamma
    TG = lambda k: t_global(machine, p, 8.0 * spec.m * k) if p > 1 else 0.0  # noqa: E731
    if method == "bicgstab":        # Eq. (14)
        return 18 * tv + 2 * ts + TG(3) + 2 * TG(1)
    if method == "ibicgstab":       # Eq. (15)
        return 20 * tv + 2 * ts + TG(7)
    if method == "pipebicgstab":    # Eq. (16)
        return 26 * tv + overlapped(ts, TG(3), g) + overlapped(ts, TG(4), g)
    if method == "pbicgstab":       # Eq. (17)
        return 19 * tv + 2 * ts + 2 * tp + TG(3) + 2 * TG(1)
    if method == "rbicgstab":       # Eq. (18)
        return 21 * tv + 2 * ts + overlapped(tp, TG(1), g) + overlapped(tp, TG(4), g)
    if method == "ppipebicgstab":   # Eq. (19)
        return 34 * tv + overlapped(ts + tp, TG(3), g) + overlapped(ts + tp, TG(4), g)
    raise ValueError(f"unknown method {method}")


def relative_performance(machine: MachineModel, spec_of, methods: Sequence[str],
                         p_range: Iterable[int], compulsory: bool = False) -> dict:
    """Sec. 4.1: R^i(p) = min_j T^j(p) / T^i(p).  spec_of(method) -> ProblemSpec
    (so the preconditioned methods can carry their alpha)."""
    out = {}
    for p in p_range:
        t = {mth: t_iteration(machine, spec_of(mth), mth, p, compulsory) for mth in methods}
        best = min(t.values())
        out[p] = {mth: best / v for mth, v in t.items()}
    return out


def speedup(times: dict) -> dict:
    """S(p) = T(1) / T(p)."""
    t1 = times[min(times)]
    return {p: t1 / t for p, t in times.items()}


def relative_speedup(times_by_method: dict, baseline: str = "bicgstab") -> dict:
    """Sec. 4.2: P^i(p) = T^baseline(p) / T^i(p)."""
    base = times_by_method[baseline]
    return {mth: {p: base[p] / t for p, t in tm.items()} for mth, tm in times_by_method.items()}


def breakeven_elements(t_g: float, b: float) -> float:
    """Eq. (21) context: Nm/p ~ T_G b / 8 (direct evaluation; the paper's printed
    2.5e4 is 10x below it, SPEC.md open question)."""
    return t_g * b / 8.0


def scan(machine: MachineModel, spec: ProblemSpec, methods: Sequence[str], p_range: Sequence[int],
         gammas: Sequence[float], alphas: Sequence[int], ms: Sequence[int]) -> list[dict]:
    """Long-form rows (method, p, gamma, alpha, m, bw_mode, T_seconds, R) -- Figs. 5-8."""
    if not methods or not p_range:
        raise ValueError("empty scan ranges")
    rows = []
    for gamma in gammas:
        mach = dataclasses.replace(machine, gamma=gamma)
        for bw_mode, bw in (("ram", machine.b), ("llc", machine.llc_b or machine.b)):
            mach_b = dataclasses.replace(mach, b=bw)
            for alpha in alphas:
                for m in ms:
                    def spec_of(mth, m=m, alpha=alpha):
                        return dataclasses.replace(spec, m=m, precond_alpha=alpha if mth in PRECONDITIONED else 0)
                    rel = relative_performance(mach_b, spec_of, methods, p_range)
                    for p in p_range:
                        for mth in methods:
                            rows.append({"method": mth, "p": p, "gamma": gamma, "alpha": alpha, "m": m,
                                         "bw_mode": bw_mode,
                                         "T_seconds": t_iteration(mach_b, spec_of(mth), mth, p),
                                         "R": rel[p][mth]})
    return rows


def _check_p(p: int) -> None:
    if p < 1:
        raise ValueError("p must be >= 1")


def fit_bandwidth(bytes_per_iteration: Sequence[float], seconds_per_iteration: Sequence[float]) -> float:
    """Least-squares b for T = Sigma / b over measured iterations (one GPU, no
    communication): b = sum(S^2) / sum(S T)."""
    num = sum(s * s for s in bytes_per_iteration)
    den = sum(s * t for s, t in zip(bytes_per_iteration, seconds_per_iteration))
    if den <= 0 or not math.isfinite(num / den):
        raise ValueError("degenerate fit")
    return num / den
