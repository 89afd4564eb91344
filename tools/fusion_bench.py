"""Fig. 2 fusion micro-benchmark on the GPU.

usage: python tools/fusion_bench.py [--n 100000000] [--reps 20]
Prints one JSON line (paper, Table 1: run1/run2 = 1.76 on CPU nodes)."""
import argparse
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_1907_12874_b200 as P  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=100_000_000)
ap.add_argument("--reps", type=int, default=20)
args = ap.parse_args()
ctx = P.Context(0)
r = P.fusion_bench(ctx, args.n, args.reps)
r["transfers"] = [9, 5, 5]
r["peak_GBps"] = json.loads((Path(__file__).resolve().parent.parent / "MEASURED_PEAKS.json").read_text())["hbm_gbs"]
print(json.dumps(r))
