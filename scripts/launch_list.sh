#!/bin/bash
# usage: bash scripts/launch_list.sh <cfg> '<opts json>' <tag>  -> gpurun_out/launches_<tag>.csv + per-kernel summary
mkdir -p gpurun_out
timeout 300 python scripts/run_once.py $1 "$2" > /dev/null 2>&1 || { echo "run_once failed"; exit 1; }
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$3.csv \
  python scripts/run_once.py $1 "$2" > /dev/null 2>&1
python - "$3" <<'PY'
import csv, sys, collections
rows = list(csv.reader(open("gpurun_out/launches_%s.csv" % sys.argv[1])))
hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h = rows[hdr]; ki, vi = h.index("Kernel Name"), h.index("Metric Value")
agg = collections.OrderedDict()
for r in rows[hdr + 1:]:
    if len(r) <= vi: continue
    name = r[ki].split("(")[0][:60]
    t = float(r[vi].replace(",", ""))
    a = agg.setdefault(name, [0, 0.0]); a[0] += 1; a[1] += t
tot = sum(v[1] for v in agg.values())
print("== %s: %d launches, %.3f ms total (per run_once: 2 calls)" % (sys.argv[1], sum(v[0] for v in agg.values()), tot / 1e6))
for k, (n, t) in agg.items():
    print("  %-60s n=%3d  %9.3f ms  %5.1f%%" % (k, n, t / 1e6, 100 * t / tot))
PY
