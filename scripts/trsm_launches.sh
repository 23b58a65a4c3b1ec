#!/bin/bash
python paper_cs_0601133_b200/build.py > /dev/null || exit 1
N=${1:-8192}
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/trsm_launches_$N.csv python scripts/run_trsm_once.py $N > /dev/null 2>&1
python - $N <<'PY'
import csv, sys, collections
rows = list(csv.reader(open("gpurun_out/trsm_launches_%s.csv" % sys.argv[1])))
h = next(i for i, r in enumerate(rows) if "Kernel Name" in r); H = rows[h]
ki, vi = H.index("Kernel Name"), H.index("Metric Value")
agg = collections.defaultdict(lambda: [0, 0.0])
for r in rows[h + 1:]:
    if len(r) <= vi: continue
    k = r[ki].split("(")[0].replace("void ", "")[:50]; agg[k][0] += 1; agg[k][1] += float(r[vi].replace(",", ""))
tot = sum(a[1] for a in agg.values())
for k, a in sorted(agg.items(), key=lambda x: -x[1][1]): print("%-52s %5d %9.3f ms %5.1f%%" % (k, a[0], a[1] / 1e6, 100 * a[1] / tot))
PY
