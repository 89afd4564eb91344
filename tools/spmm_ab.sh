#!/bin/bash
# CSR SpMM A/B on the random band of config 5 at ncu's locked base clock
# (comparable across boxes and builds).  usage: tools/spmm_ab.sh OUTDIR [m ...]
# variants: base = $MBG_LIB_BASE (another build of the library, optional),
#           nat  = natural row order (MBG_SPMM_SORT=0), sort = length-sorted twin
OUT=$1; shift
MS=${@:-8 16 32}
mkdir -p $OUT
for m in $MS; do
  for v in base nat sort; do
    case $v in
      base) [ -n "$MBG_LIB_BASE" ] || continue; ENVV="MBG_LIB=$MBG_LIB_BASE";;
      nat) ENVV="MBG_SPMM_SORT=0";;
      sort) ENVV="MBG_SPMM_SORT=1";;
    esac
    env $ENVV ncu -k regex:spmm --metrics gpu__time_duration.sum --launch-skip 4 -c 6 --csv \
        --log-file $OUT/spmm_${v}_m${m}.csv python tools/spmm_time.py --kind banded --m $m --reps 6 \
        > $OUT/spmm_${v}_m${m}.log 2>&1
    python - "$OUT/spmm_${v}_m${m}.csv" "$v" "$m" <<'PY'
import csv, io, sys
txt = open(sys.argv[1]).read()
i = txt.find('"ID"')
vals = []
for r in csv.DictReader(io.StringIO(txt[i:])):
    if r.get("Metric Name") == "gpu__time_duration.sum":
        v = float(r["Metric Value"].replace(",", ""))
        u = r.get("Metric Unit", "")
        vals.append(v / 1000.0 if u == "ns" else (v * 1000.0 if u == "ms" else v))
print(f"{sys.argv[2]:5s} m={sys.argv[3]:3s} {sum(vals)/max(1,len(vals)):9.1f} us  (n={len(vals)}, min {min(vals) if vals else 0:.1f})")
PY
  done
done
