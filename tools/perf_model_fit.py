"""Fit the paper's execution-time model on this B200 and compare it with the
measured per-iteration times.

Single GPU (no communication terms): T_iter = (V + apps*alpha) * T_vec + 2 T_mul
with V, apps from the solver's own schedule.  b is fitted by least squares
over the six methods of the C2 sweep (merged formulation) and compared with
the measured copy bandwidth; per-method predicted vs measured times are
printed for both SpMV byte models (Eq. (3) and compulsory).  Then the model
(B200 preset: measured b, ASSUMED NVLink reduction/exchange fits) gives the
relative performance R^i(p) of the six methods for C4 on p = 1..8.

usage: python tools/perf_model_fit.py [--sweep profiles/r01e_sweep_all_methods.jsonl] [--out profiles/r01h_perf_model]
"""
import argparse
import dataclasses
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import paper_1907_12874_b200 as P  # noqa: E402
from paper_1907_12874_b200 import perfmodel as M  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--sweep", default=str(ROOT / "profiles" / "r01e_sweep_all_methods.jsonl"))
ap.add_argument("--out", default=str(ROOT / "profiles" / "r01h_perf_model"))
args = ap.parse_args()

peak = json.loads((ROOT / "MEASURED_PEAKS.json").read_text())["hbm_gbs"]
rows = [json.loads(l) for l in open(args.sweep)]
c2 = [r for r in rows if r["config"] == 2 and r["formulation"] == "merged"]
N, m, nnz = 2_097_152, 8, 14_581_760
C = nnz / N
out = {"config": "C2 conv-diff 128^3 m=8, merged formulation, 1 B200", "peak_copy_GBps": peak, "models": {}}
for model in ("eq3", "compulsory"):
    comp = model == "compulsory"
    spec0 = M.ProblemSpec(N=N, m=m, C=C)
    sig = []
    meas = []
    for r in c2:
        mth = r["method"]
        s = P.method_schedule_pc(mth, "merged")
        alpha = 2 if mth in M.PRECONDITIONED else 0
        vec_bytes = (s["vec"] + s["precond"] * alpha) * 8.0 * N * m
        spmv = M.sigma_mul_compulsory(spec0) if comp else M.sigma_mul(spec0)
        sig.append(vec_bytes + 2 * spmv)
        meas.append(r["ms_per_iteration"] / 1e3)
    b = M.fit_bandwidth(sig, meas)
    mach = M.MachineModel("B200 fitted", b=b)
    per = {}
    for r, sg, t in zip(c2, sig, meas):
        mth = r["method"]
        spec = dataclasses.replace(spec0, precond_alpha=2 if mth in M.PRECONDITIONED else 0)
        pred = M.t_iteration(mach, spec, mth, 1, compulsory=comp)
        pred_peak = M.t_iteration(M.MachineModel("peak", b=peak * 1e9), spec, mth, 1, compulsory=comp)
        per[mth] = {"measured_ms": round(t * 1e3, 4), "model_fitted_b_ms": round(pred * 1e3, 4),
                    "model_peak_b_ms": round(pred_peak * 1e3, 4), "error_vs_fit": round(pred / t - 1, 4)}
    out["models"][model] = {"fitted_b_GBps": round(b / 1e9, 1), "fraction_of_copy_peak": round(b / 1e9 / peak, 3),
                            "methods": per}

# relative performance of the six methods for C4 on 1..8 B200 (strong scaling, assumed comm fits)
spec4 = M.ProblemSpec(N=320 ** 3, m=32, C=228_761_600 / 320 ** 3, halo_bytes=320 * 320 * 32 * 8)
b200 = M.b200_node(out["models"]["compulsory"]["fitted_b_GBps"], gamma=0.0)
spec_of = lambda mth: dataclasses.replace(spec4, precond_alpha=2 if mth in M.PRECONDITIONED else 0)  # noqa: E731
rel = M.relative_performance(b200, spec_of, list(M.VEC), range(1, 9), compulsory=True)
out["c4_relative_performance_p1_8"] = {"assumptions": "b fitted on C2; T_G = 10us + 0.5us l^0.21 p^0.5, "
                                       "T_L = 8us + l/450GB/s, gamma = 0 (not measured: one GPU here)",
                                       "R": {p: {k: round(v, 4) for k, v in r.items()} for p, r in rel.items()}}
# predicted parallel efficiency T(1) / (p T(p)) of C4 Pipelined (the north-star 8-GPU target)
# under the same assumed NVLink fits -- a model prediction, not a measurement
t1 = M.t_iteration(b200, spec_of("pipebicgstab"), "pipebicgstab", 1, compulsory=True)
out["c4_pipelined_predicted_efficiency"] = {
    str(p): round(t1 / (p * M.t_iteration(b200, spec_of("pipebicgstab"), "pipebicgstab", p, compulsory=True)), 4)
    for p in (1, 2, 4, 8)}
json.dump(out, open(args.out + ".json", "w"), indent=1)
lines = ["# r01h -- the paper's time model fitted on B200 (tools/perf_model_fit.py)", "",
         f"C2 conv-diff 128^3, m=8, merged formulation, one GPU; measured copy peak {peak} GB/s.", ""]
for model, d in out["models"].items():
    lines += [f"## SpMV bytes: {model} -- fitted b = {d['fitted_b_GBps']} GB/s "
              f"({100 * d['fraction_of_copy_peak']:.0f} % of the copy peak)", "",
              "| method | measured ms/it | model (fitted b) | model (copy peak) | model error |", "|---|---|---|---|---|"]
    for mth, v in d["methods"].items():
        lines.append(f"| {mth} | {v['measured_ms']} | {v['model_fitted_b_ms']} | {v['model_peak_b_ms']} | "
                     f"{100 * v['error_vs_fit']:+.1f} % |")
    lines.append("")
lines += ["## C4 (320^3, m=32) relative performance R^i(p), B200 preset (assumed comm fits)", "",
          "| p | " + " | ".join(M.VEC) + " |", "|---" * (len(M.VEC) + 1) + "|"]
for p, r in out["c4_relative_performance_p1_8"]["R"].items():
    lines.append(f"| {p} | " + " | ".join(f"{r[k]:.3f}" for k in M.VEC) + " |")
lines += ["", "## C4 Pipelined: predicted parallel efficiency T(1)/(p T(p)) (same assumed NVLink fits)", "",
          "| p | " + " | ".join(out["c4_pipelined_predicted_efficiency"]) + " |",
          "|---" * (len(out["c4_pipelined_predicted_efficiency"]) + 1) + "|",
          "| efficiency | " + " | ".join(f"{v:.3f}" for v in out["c4_pipelined_predicted_efficiency"].values()) + " |"]
open(args.out + ".md", "w").write("\n".join(lines) + "\n")
print("\n".join(lines))
