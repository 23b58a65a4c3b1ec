"""Turn raw ncu outputs from gpurun_out/ into the committed summaries under profiles/.

    python scripts/summarize_profiles.py <round> <cfg> <launches.csv> [<full.ncu-rep>]

Writes profiles/r<round>_<cfg>_launches.csv (every launch with its device time
and the step share per kernel), and, given a --set full report of the GEMM,
profiles/r<round>_<cfg>_gemm_ncu_full.txt plus profiles/ncu_gemm_<cfg>.json
(the per-launch DRAM traffic bench.py reports as roofline.traffic).
"""
import csv
import json
import os
import subprocess
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CFG_BYTES = {  # algorithmic bytes of the GEMM launch: limb planes read once + C written (+read if beta)
    "c4": 2 * 32768 * 8192 * 2 + 4 * 32768 * 32768,
}


def launches(path, out):
    lines = open(path).read().splitlines()
    start = [i for i, l in enumerate(lines) if l.startswith('"ID"')][0]
    rows = list(csv.reader(lines[start:]))
    h = rows[0]
    ki, vi, gi, bi = h.index("Kernel Name"), h.index("Metric Value"), h.index("Grid Size"), h.index("Block Size")
    res = ["id,kernel,grid,block,gpu_time_ms"]
    per = defaultdict(float)
    for r in rows[1:]:
        name = r[ki].split("(")[0].replace("void ", "").replace("ff::<unnamed>::", "")
        t = float(r[vi]) / 1e6
        res.append('%s,%s,"%s","%s",%.4f' % (r[0], name, r[gi], r[bi], t))
        if name.startswith(("ffgemm", "encode", "preadd", "scale_c")):
            per[name.split("<")[0]] += t
    tot = sum(per.values())
    res.append("# share of the library's kernel time (all launches above): " +
               "; ".join("%s %.1f%%" % (k, 100 * v / tot) for k, v in sorted(per.items(), key=lambda x: -x[1])))
    open(out, "w").write("\n".join(res) + "\n")
    print(open(out).read())


def full(rep, cfg, rnd):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(raw.splitlines()))
    h, u, v = r[0], r[1], r[2]
    want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
            "dram__throughput.avg.pct_of_peak_sustained_elapsed",
            "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
            "sm__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
            "lts__t_sectors_srcunit_tex_op_read.sum", "lts__t_sectors_srcunit_ltcfabric.sum",
            "sm__cycles_elapsed.avg.per_second", "launch__registers_per_thread", "launch__grid_size",
            "launch__block_size", "launch__shared_mem_per_block_dynamic", "launch__cluster_dim_x",
            "sm__warps_active.avg.pct_of_peak_sustained_active", "gpc__cycles_elapsed.max"]
    txt = ["# ncu --set full --clock-control none, ffgemm_tc_kernel, bench.py %s (1 GPU), round %s" % (cfg, rnd)]
    summ = {}
    for w in want:
        if w in h:
            i = h.index(w)
            summ[w] = (v[i], u[i])
            txt.append("%-70s %20s %s" % (w, v[i], u[i]))
    out = os.path.join(ROOT, "profiles", "r%s_%s_gemm_ncu_full.txt" % (rnd, cfg))
    open(out, "w").write("\n".join(txt) + "\n")
    print(open(out).read())

    def num(k):
        val, unit = summ[k]
        return float(val.replace(",", "")) * {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1,
                                              "Tbyte": 1e12}.get(unit, 1)
    traffic = num("dram__bytes_read.sum") + num("dram__bytes_write.sum")
    json.dump({"config": cfg, "world": 1, "kernel": "ffgemm_tc_kernel<2>", "round": int(rnd),
               "dram_bytes_per_launch": traffic, "dram_read_bytes": num("dram__bytes_read.sum"),
               "dram_write_bytes": num("dram__bytes_write.sum"),
               "algorithmic_bytes_per_launch": CFG_BYTES.get(cfg),
               "source": os.path.relpath(out, ROOT)},
              open(os.path.join(ROOT, "profiles", "ncu_gemm_%s.json" % cfg), "w"), indent=1)


MULTI_WANT = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
              "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
              "sm__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
              "sm__cycles_elapsed.avg.per_second", "launch__registers_per_thread", "launch__grid_size",
              "launch__cluster_dim_x", "launch__shared_mem_per_block_dynamic"]


def multi(rep, out, title):
    """Every launch of a --set full report, one block each (multi <rep> <out> <title>)."""
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(raw.splitlines()))
    h, u = r[0], r[1]
    txt = ["# " + title]
    for li, v in enumerate(r[2:]):
        txt.append("## launch %d: %s" % (li, v[h.index("Kernel Name")][:90]))
        for w in MULTI_WANT:
            if w in h:
                i = h.index(w)
                txt.append("%-70s %20s %s" % (w, v[i], u[i]))
    open(out, "w").write("\n".join(txt) + "\n")
    print(open(out).read())


if __name__ == "__main__":
    if sys.argv[1] == "multi":
        multi(sys.argv[2], sys.argv[3], sys.argv[4])
        sys.exit(0)
    rnd, cfg, lc = sys.argv[1], sys.argv[2], sys.argv[3]
    launches(lc, os.path.join(ROOT, "profiles", "r%s_%s_launches.csv" % (rnd, cfg)))
    if len(sys.argv) > 4:
        full(sys.argv[4], cfg, rnd)
