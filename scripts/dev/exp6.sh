N=${1:-2048}
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_lqup$N.csv python scripts/run_lqup_once.py $N > /dev/null 2>&1
python - $N <<'PY'
import csv, sys, collections
rows = list(csv.reader(open("gpurun_out/launches_lqup%s.csv" % sys.argv[1])))
hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h = rows[hdr]; ki, vi = h.index("Kernel Name"), h.index("Metric Value")
agg = collections.OrderedDict()
for r in rows[hdr + 1:]:
    if len(r) <= vi: continue
    name = r[ki].split("(")[0][:60]; t = float(r[vi].replace(",", ""))
    a = agg.setdefault(name, [0, 0.0]); a[0] += 1; a[1] += t
tot = sum(v[1] for v in agg.values())
print("== lqup N=%s: %d launches, GPU busy %.3f ms" % (sys.argv[1], sum(v[0] for v in agg.values()), tot / 1e6))
for k, (n, t) in agg.items(): print("  %-60s n=%4d %9.3f ms" % (k, n, t / 1e6))
PY
