"""Summarise ncu captures (.ncu-rep via `ncu -i --page raw --csv`) and launch
lists (`--metrics gpu__time_duration.sum --csv`) into profiles/.

usage: python tools/ncu_summary.py OUT.md [--launches launches.csv] [rep.ncu-rep ...]
Also writes OUT.json with per-kernel DRAM bytes (profiles/ncu_dram_bytes.json
is what bench.py reads for roofline.traffic).
"""
import csv
import io
import json
import subprocess
import sys
from collections import defaultdict

KEYS = [
    ("gpu__time_duration.sum", "us"),
    ("dram__bytes_read.sum", "dram_rd_MB"),
    ("dram__bytes_write.sum", "dram_wr_MB"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram_%"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps_active_%"),
    ("launch__registers_per_thread", "regs"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active", "fp64_pipe_%"),
    ("lts__t_sector_hit_rate.pct", "l2_hit_%"),
    ("l1tex__t_sector_hit_rate.pct", "l1_hit_%"),
]


SCALE = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
TSCALE = {"nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3, "second": 1e6}   # -> microseconds


def raw(rep):
    """Rows of the raw page; byte metrics normalised to MB using the units row."""
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        for k, u in zip(hdr, units):
            if u in SCALE and d.get(k):
                try:
                    d[k] = str(float(d[k].replace(",", "")) * SCALE[u] / 1e6)
                except ValueError:
                    pass
            elif u in TSCALE and d.get(k):
                try:
                    d[k] = str(float(d[k].replace(",", "")) * TSCALE[u])
                except ValueError:
                    pass
        res.append(d)
    return res


def launches(path):
    rows = list(csv.reader(open(path)))
    i = [k for k, r in enumerate(rows) if r and r[0] == "ID"][0]
    hdr = rows[i]
    agg = defaultdict(lambda: [0, 0.0])
    ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
    for r in rows[i + 1:]:
        n = r[ki].split("(")[0]
        agg[n][0] += 1
        agg[n][1] += float(r[vi].replace(",", ""))
    return agg


def main():
    out = sys.argv[1]
    args = sys.argv[2:]
    lines = []
    dram = {}
    if args and args[0] == "--launches":
        agg = launches(args[1])
        args = args[2:]
        tot = sum(v[1] for v in agg.values())
        lines += ["## Launch list (ncu gpu__time_duration, cold-cache, serialised)", "",
                  "| kernel | launches | total us | share |", "|---|---|---|---|"]
        for k, v in sorted(agg.items(), key=lambda kv: -kv[1][1]):
            lines.append(f"| `{k}` | {v[0]} | {v[1] / 1000:.1f} | {100 * v[1] / tot:.1f}% |")
        lines.append("")
    for rep in args:
        lines += [f"## {rep} (--set full)", "", "| kernel | " + " | ".join(k[1] for k in KEYS) + " |",
                  "|---" * (len(KEYS) + 1) + "|"]
        for d in raw(rep):
            vals = []
            for k, _ in KEYS:
                v = d.get(k, "")
                try:
                    f = float(v.replace(",", ""))
                    v = f"{f:.1f}"
                except ValueError:
                    pass
                vals.append(v)
            name = d["Kernel Name"].split("(")[0]
            lines.append(f"| `{name}` | " + " | ".join(vals) + " |")
            try:
                rd = float(d["dram__bytes_read.sum"].replace(",", ""))
                wr = float(d["dram__bytes_write.sum"].replace(",", ""))
                dram.setdefault(name, (rd + wr) * 1e6)
            except (KeyError, ValueError):
                pass
        lines.append("")
    open(out, "w").write("\n".join(lines) + "\n")
    json.dump(dram, open(out.rsplit(".", 1)[0] + ".json", "w"), indent=1)


if __name__ == "__main__":
    main()
