"""Compare per-kernel mean durations of two tools/ncu_ab.sh captures.
usage: python tools/ncu_ab_compare.py A.csv B.csv"""
import csv
import io
import sys
from collections import defaultdict


def load(path):
    txt = open(path).read()
    i = txt.find('"ID"')
    rows = list(csv.DictReader(io.StringIO(txt[i:])))
    d = defaultdict(list)
    for r in rows:
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        v = float(r["Metric Value"].replace(",", ""))
        unit = r.get("Metric Unit", "")
        v = v / 1000.0 if unit == "ns" else (v * 1000.0 if unit == "ms" else v)
        name = r["Kernel Name"].split("(")[0]
        d[name].append(v)
    return d


a, b = load(sys.argv[1]), load(sys.argv[2])
print(f"{'kernel':60s} {'n':>4s} {'A us':>9s} {'B us':>9s} {'B/A':>6s}")
for k in sorted(set(a) | set(b), key=lambda k: -sum(a.get(k, [0]))):
    ma = sum(a[k]) / len(a[k]) if k in a else float("nan")
    mb = sum(b[k]) / len(b[k]) if k in b else float("nan")
    print(f"{k[:60]:60s} {len(a.get(k, [])):4d} {ma:9.1f} {mb:9.1f} {mb / ma if ma == ma and ma else float('nan'):6.3f}")
