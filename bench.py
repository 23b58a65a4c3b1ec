#!/usr/bin/env python
"""fgemm benchmark (BASELINE.json metric: "fgemm mod-p GOPS (2mnk/s) at 1/2/4/8
B200; % tensor-pipe peak").

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c4] [--impl ours|reference]
    torchrun --nproc-per-node N ... bench.py --gpus N ...     (one process per GPU, NCCL)

A step is one whole fgemm of the chosen config (default c4: p = 65521,
m = n = 32768, k = 8192 -- the paper's prime, the config the metric's
"1/2/4/8 B200" is quoted on).  At N = 1 the step is the product's default
path, ``ff_gemm_ex`` with default options (the library picks limbs / CRT,
Winograd, the small-field kernel by itself); at N > 1 it is the row-panel
sharded path (sharded.py: B broadcast by NCCL, each rank multiplies its
panel).  Inputs are seeded synthetic matrices (ffgen recipe) already resident
in HBM; configs whose inputs fit the 126 MB L2 flush it between steps
(untimed).

Rank 0 prints ONE JSON line.  At N = 1 it also carries ``per_config``: the
other four BASELINE configs (c1, c2, c3, c5) timed the same way on the
default path.  Every timed config is verified after its timed region:
sampled output rows against the CPU oracle and Freivalds' test on the whole
output (inputs regenerated on the host by ffgen, never taken from the GPU).
``--impl reference`` times the CPU oracle (the reference arm of this tier) on a
bounded sample of the workload; it never imports the product package.
"""
from __future__ import annotations

import argparse
import importlib.util
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "fgemm mod-p GOPS (2mnk/s) at 1/2/4/8 B200; % tensor-pipe peak"
L2_BYTES = 126 * 2 ** 20


def _load_configs():
    """configs.py is pure data; load it by path so that the reference arm never
    imports the product package (whose __init__ maps libffgemm.so)."""
    spec = importlib.util.spec_from_file_location(
        "_ff_configs", os.path.join(ROOT, "paper_cs_0601133_b200", "configs.py"))
    mod = importlib.util.module_from_spec(spec)
    sys.modules["_ff_configs"] = mod
    spec.loader.exec_module(mod)
    return mod.CONFIGS


def _env_int(name, default):
    try:
        return int(os.environ.get(name, default))
    except ValueError:
        return default


def _peaks():
    """int8 tensor peak (TOPS) = measured bf16 x 2 (the guide's nominal int8:bf16 =
    fp8:bf16 = 4.5:2.25 POPS), from the driver-written MEASURED_PEAKS.json."""
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            mp = json.load(f)
        return {"burst": 2 * mp["bf16_tflops"], "sustained": 2 * mp["bf16_tflops_sustained"],
                "hbm_gbs": mp["hbm_gbs"], "source": "MEASURED_PEAKS.json (measured bf16 x 2)"}
    except Exception:
        return {"burst": 2 * 1590.0, "sustained": 2 * 1400.0, "hbm_gbs": 6650.0,
                "source": "fallback of B200_PROFILING.md (bf16 x 2)"}


# ------------------------------------------------------------------ clocks

class ClockSampler:
    """nvidia-smi sampled every 100 ms during the timed region (B200_PROFILING.md recipe)."""
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index):
        self.gpu = gpu_index
        self.proc = None
        self.rows = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), "--query-gpu=" + self.Q,
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *a):
        self.rows = []
        if self.proc is not None:
            self.proc.terminate()
            try:
                out, _ = self.proc.communicate(timeout=5)
            except Exception:
                self.proc.kill()
                out = ""
            for line in out.strip().splitlines():
                parts = [x.strip() for x in line.split(",")]
                if len(parts) >= 9:
                    self.rows.append(parts)
        return False

    def summary(self):
        rows = self.rows
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"], "samples": 0}
        num = lambda s: s.replace(".", "").isdigit()  # noqa: E731
        sm = [float(r[1]) for r in rows if num(r[1])]
        mx = [float(r[2]) for r in rows if num(r[2])]
        pw = [float(r[3]) for r in rows if num(r[3])]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[5 + i].lower().startswith("active")})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(rows), "power_w_max": max(pw) if pw else None}


# ------------------------------------------------------------------ CPU oracle (baseline / reference arm)

def _host_inputs_for_oracle(cfg, rows):
    """Host copies from the ffgen recipe (never from the CUDA path): the sampled
    rows of op(A) (as a stored array + row ids) and all of B."""
    import numpy as np
    import ffgen
    if cfg.transA == "N":
        A = np.zeros((cfg.m, cfg.k), dtype=np.int32)  # only sampled rows are filled / read
        for r in rows:
            A[r] = ffgen.uniform_matrix(cfg.p, cfg.seed, ffgen.STREAM_A, cfg.m, cfg.k, row0=r, nrows=1)[0]
    else:
        A = ffgen.uniform_matrix(cfg.p, cfg.seed, ffgen.STREAM_A, cfg.k, cfg.m)
    B = ffgen.uniform_matrix(cfg.p, cfg.seed, ffgen.STREAM_B, *cfg.b_shape)
    Cin = None
    if cfg.beta % cfg.p:
        Cin = np.stack([ffgen.uniform_matrix(cfg.p, cfg.seed, ffgen.STREAM_C, cfg.m, cfg.n, row0=r, nrows=1)[0]
                        for r in rows])
    return A, B, Cin


def _oracle_rows_timed(cfg, rows, A, B, Cin, threads):
    import oracle
    t0 = time.perf_counter()
    oracle.fgemm_rows(cfg.p, cfg.transA, cfg.transB, cfg.alpha, A, B, cfg.beta, Cin, rows,
                      cfg.m, cfg.n, cfg.k, nthreads=threads)
    return time.perf_counter() - t0


def cpu_oracle_sample(cfg, target_s=12.0, max_rows=256):
    """Time the oracle, as it stands, on a bounded sample: whole output rows of
    the config (each a full length-k dot product with every column)."""
    import oracle
    oracle.build()
    threads = len(os.sched_getaffinity(0))
    rows_all = list(range(0, cfg.m, max(1, cfg.m // max_rows)))[:max_rows]
    A, B, Cin_all = _host_inputs_for_oracle(cfg, rows_all)
    t1 = _oracle_rows_timed(cfg, rows_all[:1], A, B, None if Cin_all is None else Cin_all[:1], threads)
    nrows = int(max(1, min(len(rows_all), round(target_s / max(t1, 1e-6)))))
    rows = rows_all[:nrows]
    t = _oracle_rows_timed(cfg, rows, A, B, None if Cin_all is None else Cin_all[:nrows], threads)
    gops = 2.0 * nrows * cfg.n * cfg.k / t / 1e9
    return {"value": gops, "unit": "GOPS", "cores": threads, "kind": "oracle",
            "sample": "%d full output rows of %s (%d x %d x k=%d each), %.1f s" % (
                nrows, cfg.name, 1, cfg.n, cfg.k, t),
            "cpu": _cpu_model()}, (rows_all, A, B, Cin_all, threads)


def _cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return None


def _mapped_product_libs():
    """Product shared objects mapped into this process (the reference arm must have none)."""
    try:
        with open("/proc/self/maps") as f:
            return sorted({ln.split()[-1] for ln in f if "libffgemm" in ln})
    except OSError:
        return []


def run_reference(args, cfg):
    rank = _env_int("RANK", 0)
    if rank != 0:
        return 0       # the reference arm is the CPU oracle: rank 0 alone runs it
    world = _env_int("WORLD_SIZE", 1)
    base, (rows_all, A, B, Cin_all, threads) = cpu_oracle_sample(cfg, target_s=4.0)
    nrows = int(base["sample"].split()[0])
    times = []
    for i in range(args.warmup + args.steps):
        t = _oracle_rows_timed(cfg, rows_all[:nrows], A, B,
                               None if Cin_all is None else Cin_all[:nrows], threads)
        if i >= args.warmup:
            times.append(t)
    tot = sum(times)
    value = 2.0 * nrows * cfg.n * cfg.k * len(times) / tot / 1e9
    leaked = _mapped_product_libs()
    if leaked:
        raise SystemExit("reference arm: the product library is mapped into this process: %s" % leaked)
    line = {
        "metric": METRIC, "value": value, "unit": "GOPS", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1e3 * tot / len(times), "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "int64/int128", "data": "synthetic",
        "impl": "reference",
        "config": _config_json(cfg, world, ref_rows=nrows),
        "cpu_baseline": {"value": value, "unit": "GOPS", "cores": threads, "kind": "oracle",
                         "sample": "each step: %d full output rows of %s (1 x %d x k=%d each)" % (
                             nrows, cfg.name, cfg.n, cfg.k), "cpu": _cpu_model()},
        "e2e": {"value": value, "unit": "GOPS", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "product_libs_mapped": leaked,
    }
    print(json.dumps(line), flush=True)
    return 0


def _config_json(cfg, world, **extra):
    d = {"workload": cfg.name + ": " + cfg.text, "p": cfg.p, "m": cfg.m, "n": cfg.n, "k": cfg.k,
         "transA": cfg.transA, "transB": cfg.transB, "alpha": cfg.alpha, "beta": cfg.beta,
         "seed": cfg.seed, "parallelism": "row-panel x%d, B broadcast (NCCL)" % world if world > 1
         else "single GPU"}
    d.update(extra)
    return d


# ------------------------------------------------------------------ verification (CPU oracle)

def verify_output(cfg, C_out, row0=0, nsample=8, trials=2):
    """Check rows [row0, row0 + C_out.shape[0]) of the config's output (host int32
    numpy) against the CPU oracle on inputs regenerated by ffgen: `nsample`
    sampled rows bit-exactly, and Freivalds' test on the whole block
    (C_out x == alpha op(A)(op(B) x) + beta C_in x mod p, `trials` random x;
    a wrong block passes one trial with probability <= 1/p)."""
    import numpy as np
    import ffgen
    import oracle
    t0 = time.perf_counter()
    # torchrun sets OMP_NUM_THREADS=1: give each local rank its share of the host cores
    nth = max(1, len(os.sched_getaffinity(0)) // max(1, _env_int("LOCAL_WORLD_SIZE", 1)))
    ffgen.set_threads(nth)
    p, mr = cfg.p, C_out.shape[0]
    if cfg.transA == "N":
        A_rows = ffgen.uniform_matrix(p, cfg.seed, ffgen.STREAM_A, *cfg.a_shape, row0=row0, nrows=mr)
    else:
        A_rows = ffgen.uniform_matrix(p, cfg.seed, ffgen.STREAM_A, *cfg.a_shape)[:, row0:row0 + mr]
    B = ffgen.uniform_matrix(p, cfg.seed, ffgen.STREAM_B, *cfg.b_shape)
    beta_nz = cfg.beta % p != 0
    Cin = ffgen.uniform_matrix(p, cfg.seed, ffgen.STREAM_C, cfg.m, cfg.n, row0=row0, nrows=mr) if beta_nz else None
    rows = sorted({0, mr - 1} | {int(r) for r in np.linspace(0, mr - 1, nsample).astype(int)})
    want = oracle.fgemm_rows(p, cfg.transA, cfg.transB, cfg.alpha, A_rows, B, cfg.beta,
                             None if Cin is None else Cin[rows], rows, mr, cfg.n, cfg.k, nthreads=nth)
    rows_ok = bool(np.array_equal(C_out[rows], want))
    frei_ok = True
    for t in range(trials):
        x = ffgen.uniform_vector(p, cfg.seed, 8 + t, cfg.n)
        lhs = oracle.matvec(p, "N", C_out, x, nthreads=nth)
        bx = oracle.matvec(p, cfg.transB, B, x, nthreads=nth)
        rhs = oracle.matvec(p, cfg.transA, A_rows, bx, nthreads=nth).astype(np.int64) * (cfg.alpha % p) % p
        if Cin is not None:
            rhs = (rhs + oracle.matvec(p, "N", Cin, x, nthreads=nth).astype(np.int64) * (cfg.beta % p)) % p
        frei_ok = frei_ok and bool(np.array_equal(lhs.astype(np.int64), rhs))
    return {"ok": rows_ok and frei_ok, "rows_checked": len(rows), "rows_bitexact": rows_ok,
            "freivalds_trials": trials, "freivalds_ok": frei_ok, "rows": [row0, row0 + mr],
            "seconds": round(time.perf_counter() - t0, 2)}


# ------------------------------------------------------------------ GPU arm: one config on one GPU

class SingleGpu:
    """The product's default path on one GPU: ff_gemm_ex with default options and
    a caller workspace, on torch's current stream."""

    def __init__(self, ff, cfg, dev):
        import torch
        import ffgen
        self.ff, self.cfg, self.dev, self.torch = ff, cfg, dev, torch
        self.A = torch.empty(cfg.a_shape, dtype=torch.int32, device=dev)
        ff.ff_fill_uniform(self.A, *cfg.a_shape, cfg.a_shape[1], cfg.p, cfg.seed, ffgen.STREAM_A)
        self.B = torch.empty(cfg.b_shape, dtype=torch.int32, device=dev)
        ff.ff_fill_uniform(self.B, *cfg.b_shape, cfg.b_shape[1], cfg.p, cfg.seed, ffgen.STREAM_B)
        self.C = torch.zeros((cfg.m, cfg.n), dtype=torch.int32, device=dev)
        self.reset_c()
        self.ws_bytes = ff.ff_gemm_workspace_size(cfg.p, cfg.transA, cfg.transB, cfg.m, cfg.n, cfg.k)
        self.ws = torch.empty(max(1, self.ws_bytes), dtype=torch.uint8, device=dev)
        self.launches_per_step = None

    def reset_c(self):
        import ffgen
        cfg = self.cfg
        if cfg.beta % cfg.p:
            self.ff.ff_fill_uniform(self.C, cfg.m, cfg.n, cfg.n, cfg.p, cfg.seed, ffgen.STREAM_C)

    def step(self):
        cfg, A, B, C = self.cfg, self.A, self.B, self.C
        self.ff.ff_gemm_ex(cfg.p, cfg.transA, cfg.transB, cfg.m, cfg.n, cfg.k, cfg.alpha, A, A.stride(0),
                           B, B.stride(0), cfg.beta, C, C.stride(0), None, self.ws, self.ws_bytes)

    def free(self):
        self.A = self.B = self.C = self.ws = None


def _products(ff, cfg):
    """int8 products per output entry (limb pairs L^2 or CRT moduli)."""
    info = ff.ff_plan_query(cfg.p, cfg.k)
    return (info["L"] if info["scheme"] == "CRT" else info["L"] ** 2), info


def time_steps(ff, step, steps, warmup, flush_buf=None, barrier=None, prof_cap=4096):
    """Warm up, then time `steps` steps with CUDA events on torch's current stream
    (the stream every library launch of the step goes to), recording the
    library's GEMM-kernel launches with ff_prof (events on the same stream)."""
    import torch
    for _ in range(warmup):
        step()
    torch.cuda.synchronize()
    if barrier:
        barrier()
    torch.cuda.synchronize()
    cur = torch.cuda.current_stream()
    ff.ff_prof_start(prof_cap)
    if flush_buf is None:
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(cur)
        for _ in range(steps):
            step()
        e1.record(cur)
        torch.cuda.synchronize()
        elapsed = e0.elapsed_time(e1)
    else:
        elapsed = 0.0
        for _ in range(steps):
            flush_buf.fill_(1)                     # L2 flush (a buffer larger than L2), untimed
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(cur)
            step()
            e1.record(cur)
            torch.cuda.synchronize()
            elapsed += e0.elapsed_time(e1)
    gemm_ms, launches = ff.ff_prof_stop(prof_cap)
    return elapsed, gemm_ms, launches


def roofline_entry(peaks, ops_per_launch, gemm_ms, elapsed_ms, kernel):
    avg = statistics.mean(gemm_ms) if gemm_ms else float("nan")
    ach = ops_per_launch / (avg / 1e3) / 1e12 if gemm_ms else float("nan")
    return {"bound": "tensor", "achieved": ach, "peak": peaks["burst"], "unit": "TFLOP/s",
            "frac": ach / peaks["burst"], "kernel": kernel, "ops_per_launch": ops_per_launch,
            "avg_launch_ms": avg, "gemm_launches": len(gemm_ms),
            "gemm_share_of_step": sum(gemm_ms) / elapsed_ms if elapsed_ms else None,
            "peak_source": peaks["source"] + ", burst figure",
            "frac_of_sustained_peak": ach / peaks["sustained"]}


def _kernel_name(ff, cfg, launches_per_step, launches_total_per_step):
    info = ff.ff_plan_query(cfg.p, cfg.k)
    if launches_total_per_step == 1 and cfg.p < 65536:
        return "lat_gemm_kernel (tcgen05.mma.kind::i8 byte products, split-K cluster, p < 2^16 latency path)"
    wino = " x7 (one Winograd level)" if launches_per_step == 7 else ""
    return "ffgemm_tc_kernel (tcgen05.mma.kind::i8, %s)%s" % (info["scheme"], wino)


def bench_single_config(ff, cfg, steps, warmup, peaks, dev, verify=True, with_clocks=False, local=0):
    """Time one config on the default path; returns its per-config record."""
    import torch
    eng = SingleGpu(ff, cfg, dev)
    in_bytes = 4 * (cfg.m * cfg.k + cfg.k * cfg.n + (cfg.m * cfg.n if cfg.beta % cfg.p else 0))
    flush = in_bytes < 2 * L2_BYTES
    scratch = torch.empty(2 * L2_BYTES // 4, dtype=torch.int32, device=dev) if flush else None
    torch.cuda.synchronize()
    clk = ClockSampler(local) if with_clocks else None
    if clk:
        clk.__enter__()
    elapsed, gemm_ms, launches = time_steps(ff, eng.step, steps, warmup, scratch)
    if clk:
        clk.__exit__()
    prods, info = _products(ff, cfg)
    n_gemm = max(1, len(gemm_ms) // steps)
    wino = n_gemm == 7
    ops_step = prods * 2.0 * cfg.m * cfg.n * cfg.k * (7.0 / 8.0 if wino else 1.0)
    ms = elapsed / steps
    rec = {"config": cfg.name, "workload": cfg.text, "ms_per_step": ms,
           "value": cfg.useful_ops() / (ms / 1e3) / 1e9, "unit": "GOPS",
           "scheme": info["scheme"], "planes": info["L"], "int8_products_per_output": prods,
           "winograd": wino, "gpu_launches_per_step": launches / steps,
           "mma_ops_per_step": ops_step,
           "tensor_frac_of_step": ops_step / (ms / 1e3) / 1e12 / peaks["burst"],
           "l2": "flushed between steps (inputs < 2 x L2)" if flush else "inputs larger than L2 (no flush)",
           "roofline": roofline_entry(peaks, ops_step / n_gemm, gemm_ms, elapsed,
                                      _kernel_name(ff, cfg, n_gemm, launches / steps))}
    if clk:
        rec["clocks"] = clk.summary()
        if rec["clocks"].get("samples", 0) < 3:
            # a short timed region: sample the clocks over ~0.6 s of the same steps (untimed)
            with ClockSampler(local) as clk2:
                time.sleep(0.3)
                t_end = time.perf_counter() + 0.6
                while time.perf_counter() < t_end:
                    for _ in range(20):
                        eng.step()
                    torch.cuda.synchronize()
            rec["clocks"] = dict(clk2.summary(), window="0.6 s of repeated steps after the timed region")
    if ms < 0.2:
        # launch-bound: the same call captured once in a CUDA graph and replayed, so
        # the host's enqueue cost (Python + C ABI + launch) is out of the timed
        # region; still L2-flushed before every replay, device events around it
        rec["graph"] = graph_step_time(eng, steps, scratch)
    if verify:
        eng.reset_c()
        eng.step()
        torch.cuda.synchronize()
        rec["verify"] = verify_output(cfg, eng.C.cpu().numpy())
    eng.free()
    del scratch
    torch.cuda.empty_cache()
    return rec, (elapsed, gemm_ms, launches, eng)


def graph_step_time(eng, steps, flush_buf):
    """Device time of one step replayed from a CUDA graph (captured after warm-up)."""
    import torch
    cur = torch.cuda.current_stream()
    side = torch.cuda.Stream()
    side.wait_stream(cur)
    with torch.cuda.stream(side):
        eng.step()                       # workspace and function attributes settled before capture
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        eng.step()
    torch.cuda.synchronize()
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    total = 0.0
    for _ in range(steps):
        if flush_buf is not None:
            flush_buf.fill_(1)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(cur)
        g.replay()
        e1.record(cur)
        torch.cuda.synchronize()
        total += e0.elapsed_time(e1)
    del g
    return {"ms_per_step": total / steps, "steps": steps,
            "how": "the ff_gemm_ex call captured in a CUDA graph, replayed once per step; L2 flushed "
                   "before each replay; CUDA events around the replay"}


# ------------------------------------------------------------------ main

def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="c4")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--chunks", type=int, default=4, help="B column chunks broadcast when N > 1")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-verify", action="store_true")
    ap.add_argument("--no-per-config", action="store_true")
    ap.add_argument("--per-config-steps", type=int, default=10)
    args = ap.parse_args()
    args.warmup = max(3, args.warmup)

    CONFIGS = _load_configs()
    cfg = CONFIGS[args.config]
    if args.impl == "reference":
        return run_reference(args, cfg)

    import torch
    import torch.distributed as dist

    world = _env_int("WORLD_SIZE", 1)
    rank = _env_int("RANK", 0)
    local = _env_int("LOCAL_RANK", 0)
    # FF_BENCH_SHARE_GPU=1 (testing only): every rank on cuda:0 over gloo, to run
    # this multi-rank code path on a 1-GPU box; the real path is NCCL, one GPU per rank.
    share = os.environ.get("FF_BENCH_SHARE_GPU") == "1"
    if share:
        local = 0
    torch.cuda.set_device(local)
    if world > 1:
        if share:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    import paper_cs_0601133_b200 as ff
    dev = torch.device("cuda", local)
    peaks = _peaks()

    def barrier():
        if world > 1:
            if share:
                dist.barrier()
            else:
                dist.barrier(device_ids=[local])

    prods, info = _products(ff, cfg)
    verify = None
    if world == 1:
        # ---- N = 1: the default path, ff_gemm_ex
        with ClockSampler(local) as clk:
            rec, (elapsed_ms, gemm_ms, launches, eng) = bench_single_config(
                ff, cfg, args.steps, args.warmup, peaks, dev, verify=False)
        e2e_eng = None
        row0, mr = 0, cfg.m
        roofline = rec["roofline"]
        flush_note = rec["l2"]
        chunks = 1
        parallelism_extra = {"path": "ff_gemm_ex, default options"}
        if not args.no_verify:
            eng = SingleGpu(ff, cfg, dev)
            eng.step()
            torch.cuda.synchronize()
            verify = verify_output(cfg, eng.C.cpu().numpy())
            eng.free()
            torch.cuda.empty_cache()
    else:
        # ---- N > 1: row-panel sharding (sharded.py)
        from paper_cs_0601133_b200.sharded import Problem, RowPanelGemm
        import ffgen
        prob = Problem(cfg.p, cfg.m, cfg.n, cfg.k, cfg.transA, cfg.transB, cfg.alpha, cfg.beta)
        eng = RowPanelGemm(prob, chunks=args.chunks)
        r0, r1 = eng.row0, eng.row1
        row0, mr = r0, r1 - r0
        if cfg.transA == "N":
            A_panel = torch.empty((max(mr, 1), cfg.k), dtype=torch.int32, device=dev)
            ff.ff_fill_uniform(A_panel, mr, cfg.k, cfg.k, cfg.p, cfg.seed, ffgen.STREAM_A, index0=r0 * cfg.k)
        else:
            A_full = torch.empty(cfg.a_shape, dtype=torch.int32, device=dev)
            ff.ff_fill_uniform(A_full, *cfg.a_shape, cfg.a_shape[1], cfg.p, cfg.seed, ffgen.STREAM_A)
            A_panel = A_full[:, r0:r1]
        B = None
        if rank == 0:
            B = torch.empty(cfg.b_shape, dtype=torch.int32, device=dev)
            ff.ff_fill_uniform(B, *cfg.b_shape, cfg.b_shape[1], cfg.p, cfg.seed, ffgen.STREAM_B)
        C_panel = torch.zeros((max(mr, 1), cfg.n), dtype=torch.int32, device=dev)

        def reset_c():
            if cfg.beta % cfg.p:
                ff.ff_fill_uniform(C_panel, mr, cfg.n, cfg.n, cfg.p, cfg.seed, ffgen.STREAM_C, index0=r0 * cfg.n)
        reset_c()
        in_bytes = 4 * (cfg.m * cfg.k + cfg.k * cfg.n)
        flush = in_bytes < 2 * L2_BYTES
        scratch = torch.empty(2 * L2_BYTES // 4, dtype=torch.int32, device=dev) if flush else None
        flush_note = "flushed between steps (inputs < L2)" if flush else "inputs larger than L2 (no flush)"
        torch.cuda.synchronize()
        with ClockSampler(local) as clk:
            elapsed_ms, gemm_ms, launches = time_steps(
                ff, lambda: eng.step(A_panel, B, C_panel), args.steps, args.warmup, scratch, barrier)
        chunks = len(eng.chunks)
        n_gemm = max(1, len(gemm_ms) // args.steps)
        wino = eng.whole and n_gemm == 7
        ops_step = prods * 2.0 * mr * cfg.n * cfg.k * (7.0 / 8.0 if wino else 1.0)
        roofline = roofline_entry(peaks, ops_step / n_gemm, gemm_ms, elapsed_ms,
                                  "ffgemm_tc_kernel (tcgen05.mma.kind::i8, %s)%s" % (
                                      info["scheme"], " x7 (one Winograd level per panel)" if wino else ""))
        path = {"planes": "RowPanelGemm: encoded B planes broadcast (NCCL), ff_encode + ff_gemm_limbs per chunk",
                "int32": "RowPanelGemm: int32 B broadcast (NCCL), per-rank encode + ff_gemm_limbs per chunk"}[eng.mode]
        if eng.whole:
            path = "RowPanelGemm: int32 B broadcast (NCCL), one ff_gemm_ex per panel (local Winograd)"
        parallelism_extra = {"path": path, "rank_rows": [r0, r1], "broadcast_mode": eng.mode}
        if not args.no_verify:
            reset_c()
            eng.step(A_panel, B, C_panel)
            torch.cuda.synchronize()
            verify = verify_output(cfg, C_panel[:mr].cpu().numpy(), row0=r0)
        e2e_eng = (eng, A_panel, B, C_panel)

    # max over ranks of the device time
    t = torch.tensor([elapsed_ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    elapsed_ms = float(t.item())
    ms_per_step = elapsed_ms / args.steps
    value = cfg.useful_ops() * args.steps / (elapsed_ms / 1e3) / 1e9      # GOPS, whole job
    ok = torch.tensor([1 if (verify is None or verify["ok"]) else 0], dtype=torch.int32, device=dev)
    if world > 1:
        dist.all_reduce(ok, op=dist.ReduceOp.MIN)

    traffic = None
    prof = os.path.join(ROOT, "profiles", "ncu_gemm_%s.json" % cfg.name)
    if os.path.exists(prof):
        try:
            with open(prof) as f:
                pj = json.load(f)
            if pj.get("world", 1) == world:
                traffic = pj.get("dram_bytes_per_launch")
                roofline["traffic_source"] = "profiles/ncu_gemm_%s.json (ncu --set full, one launch)" % cfg.name
        except Exception:
            traffic = None
    roofline["traffic"] = traffic

    # clock-normalised tensor peak: 16384 int8 ops/clk/SM (one
    # 256x256x32 CTA-pair MMA per 128 cycles) at the median SM clock sampled
    # during the timed region
    clocks = clk.summary()
    nsm = torch.cuda.get_device_properties(dev).multi_processor_count
    if clocks.get("sm_mhz"):
        roofline["clock_peak"] = nsm * 16384 * clocks["sm_mhz"] * 1e6 / 1e12
        roofline["frac_of_clock_peak"] = roofline["achieved"] / roofline["clock_peak"]

    # measured int8 ceilings on this box: tcgen05 MMA-only loop, torch._int_mm
    if rank == 0 and world == 1:
        roofline["int8_ceilings"] = measure_int8_ceilings(ff, dev)

    # ---- the other BASELINE configs on the default path (N = 1)
    per_config = None
    if rank == 0 and world == 1 and not args.no_per_config:
        per_config = {}
        for name, c in CONFIGS.items():
            if name == cfg.name:
                continue
            st = args.per_config_steps if c.useful_ops() < 1e13 else max(3, args.per_config_steps // 2)
            r, _ = bench_single_config(ff, c, st, args.warmup, peaks, dev, verify=not args.no_verify,
                                       with_clocks=True, local=local)
            per_config[name] = r

    # ---- end to end through the public API with host buffers
    e2e = None
    if not args.no_e2e:
        e2e = run_e2e(args, cfg, ff, world, rank, local, dev, e2e_eng)

    # ---- CPU baseline: the oracle on host cores (rank 0, N = 1 only)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        cpu, _ = cpu_oracle_sample(cfg)

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "GOPS", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "int8",
            "data": "synthetic: seeded uniform residues in [0,p) (ffgen splitmix64 recipe), int32 in HBM",
            "config": _config_json(cfg, world, limbs=info["L"], scheme=info["scheme"], kb=info["kb"],
                                   chunks=chunks, l2=flush_note, **parallelism_extra),
            "tensor_pipe_pct": 100.0 * prods * cfg.useful_ops() * args.steps / (elapsed_ms / 1e3) / 1e12
            / (world * peaks["burst"]),
            "roofline": roofline,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": launches,
            "gemm_launches": len(gemm_ms),
            "clocks": clocks,
            "verify": dict(verify or {}, all_ranks_ok=bool(ok.item())) if not args.no_verify else None,
            "per_config": per_config,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    if not args.no_verify and not bool(ok.item()):
        return 1
    return 0


def measure_int8_ceilings(ff, dev):
    """The int8 MMA ceiling measured on this box: the library's tcgen05 MMA-only
    loop (SMEM-resident operands, no epilogue; ff_mma_ceiling) and cuBLASLt's
    int8 GEMM through torch._int_mm at 8192^3 (best of 10)."""
    import torch
    out = {}
    try:
        out["tcgen05_mma_only_tops"] = ff.ff_mma_ceiling()
    except Exception as e:  # pragma: no cover - informational
        out["tcgen05_mma_only_tops"] = None
        out["tcgen05_error"] = str(e)[:200]
    try:
        a = torch.randint(-128, 127, (8192, 8192), dtype=torch.int8, device=dev)
        b = torch.randint(-128, 127, (8192, 8192), dtype=torch.int8, device=dev).t()
        for _ in range(3):
            torch._int_mm(a, b)
        torch.cuda.synchronize()
        best = 1e9
        for _ in range(10):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            torch._int_mm(a, b)
            e1.record()
            torch.cuda.synchronize()
            best = min(best, e0.elapsed_time(e1))
        out["torch_int_mm_8192_tops"] = 2 * 8192 ** 3 / (best / 1e3) / 1e12
        del a, b
    except Exception as e:  # pragma: no cover
        out["torch_int_mm_8192_tops"] = None
        out["int_mm_error"] = str(e)[:200]
    torch.cuda.empty_cache()
    return out


def run_e2e(args, cfg, ff, world, rank, local, dev, sharded):
    """Same metric through the public API with pinned HOST buffers: each step
    copies the inputs host->device and the result device->host (timed)."""
    import torch
    import torch.distributed as dist
    import ffgen

    beta_nz = cfg.beta % cfg.p != 0
    steps = max(1, min(args.steps, 5))
    if world == 1:
        hA = torch.from_numpy(ffgen.uniform_matrix(cfg.p, cfg.seed, ffgen.STREAM_A, *cfg.a_shape)).pin_memory()
        hB = torch.from_numpy(ffgen.uniform_matrix(cfg.p, cfg.seed, ffgen.STREAM_B, *cfg.b_shape)).pin_memory()
        hC = torch.zeros((cfg.m, cfg.n), dtype=torch.int32).pin_memory()
    else:
        eng, A_panel, B, C_panel = sharded
        hA = torch.empty(A_panel.shape, dtype=torch.int32, pin_memory=True)
        hA.copy_(A_panel)
        hB = None
        if rank == 0:
            hB = torch.empty(B.shape, dtype=torch.int32, pin_memory=True)
            hB.copy_(B)
        hC = torch.empty(C_panel.shape, dtype=torch.int32, pin_memory=True)
        hC.copy_(C_panel)
    torch.cuda.synchronize()

    def one_step():
        if world == 1:
            # the C-ABI host entry point: copies in, computes, copies back, synchronises
            ff.ff_gemm_host(cfg.p, cfg.transA, cfg.transB, cfg.m, cfg.n, cfg.k, cfg.alpha, hA.data_ptr(),
                            hA.stride(0), hB.data_ptr(), hB.stride(0), cfg.beta, hC.data_ptr(), hC.stride(0))
        else:
            A_panel.copy_(hA, non_blocking=True)
            if rank == 0:
                B.copy_(hB, non_blocking=True)
            if beta_nz:
                C_panel.copy_(hC, non_blocking=True)
            eng.step(A_panel, B, C_panel)
            hC.copy_(C_panel, non_blocking=True)
            torch.cuda.current_stream().synchronize()

    for _ in range(max(1, min(args.warmup, 2))):
        one_step()
    if world > 1:
        if os.environ.get("FF_BENCH_SHARE_GPU") == "1":
            dist.barrier()
        else:
            dist.barrier(device_ids=[local])
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        one_step()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)                 # device clock (legacy default stream)
    t = torch.tensor([ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item())
    checked = None
    if world == 1 and not beta_nz and not args.no_verify:
        checked = verify_output(cfg, hC.numpy(), nsample=4, trials=1)
    a_bytes = 4 * cfg.m * cfg.k
    h2d = a_bytes + 4 * cfg.k * cfg.n + (4 * cfg.m * cfg.n if beta_nz else 0)
    d2h = 4 * cfg.m * cfg.n
    return {"value": cfg.useful_ops() * steps / (ms / 1e3) / 1e9, "unit": "GOPS", "steps": steps,
            "ms_per_step": ms / steps, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
            "api": "ff_gemm_host (C ABI, pinned host buffers)" if world == 1 else
            "RowPanelGemm.step with pinned host<->device copies per rank",
            "verify": checked}


if __name__ == "__main__":
    sys.exit(main())
