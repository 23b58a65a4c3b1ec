#!/usr/bin/env python
"""fgemm benchmark (BASELINE.json metric: "fgemm mod-p GOPS (2mnk/s) at 1/2/4/8
B200; % tensor-pipe peak").

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c4] [--impl ours|reference]
    torchrun --nproc-per-node N ... bench.py --gpus N ...     (one process per GPU, NCCL)

A step is one whole fgemm of the chosen config (default c4: p = 65521,
m = n = 32768, k = 8192 -- the paper's prime, row-panel sharded over 1/2/4/8 GPUs):
encode(B) [+ NCCL broadcast of B's limbs], encode(A panel), tcgen05 limb GEMM
with the fused mod-p epilogue.  Inputs are seeded synthetic matrices (ffgen
recipe) already resident in HBM; they are larger than the 126 MB L2, so no
flush is needed between steps (configs whose inputs fit in L2 flush it,
untimed).  Rank 0 prints ONE JSON line.  `--impl reference` times the CPU
oracle (the reference arm of this tier) on a bounded sample of the workload.
"""
from __future__ import annotations

import argparse
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


def _env_int(name, default):
    try:
        return int(os.environ.get(name, default))
    except ValueError:
        return default


def _peaks():
    """int8 tensor peak (TOPS) = measured bf16 x 2 (nominal int8:bf16 = 4.5:2.25 POPS)."""
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
    """nvidia-smi sampled every 200 ms during the timed region (B200_PROFILING.md recipe)."""
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index):
        self.gpu = gpu_index
        self.proc = None

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
        rows = getattr(self, "rows", [])
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"], "samples": 0}
        sm = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[5 + i].lower().startswith("active")})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(rows),
                "power_w_max": max(float(r[3]) for r in rows if r[3].replace(".", "").isdigit())
                if any(r[3].replace(".", "").isdigit() for r in rows) else None}


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
    }
    print(json.dumps(line), flush=True)
    return 0


def _config_json(cfg, world, **extra):
    d = {"workload": cfg.name + ": " + cfg.text, "p": cfg.p, "m": cfg.m, "n": cfg.n, "k": cfg.k,
         "transA": cfg.transA, "transB": cfg.transB, "alpha": cfg.alpha, "beta": cfg.beta,
         "seed": cfg.seed, "parallelism": "row-panel x%d, B limbs broadcast (NCCL)" % world if world > 1
         else "single GPU"}
    d.update(extra)
    return d


# ------------------------------------------------------------------ GPU arm

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
    args = ap.parse_args()

    from paper_cs_0601133_b200.configs import CONFIGS
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
    import ffgen
    import paper_cs_0601133_b200 as ff
    from paper_cs_0601133_b200.sharded import Problem, RowPanelGemm

    prob = Problem(cfg.p, cfg.m, cfg.n, cfg.k, cfg.transA, cfg.transB, cfg.alpha, cfg.beta)
    eng = RowPanelGemm(prob, chunks=args.chunks)
    info = ff.ff_plan_query(cfg.p, cfg.k)
    L = info["L"]
    prods = L if info["scheme"] == "CRT" else L * L       # int8 products per output (limb pairs or moduli)
    dev = torch.device("cuda", local)

    # ---- inputs, generated on device (seeded, ffgen recipe; the tests check the twin)
    r0, r1 = eng.row0, eng.row1
    mr = r1 - r0
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
    if cfg.beta % cfg.p:
        ff.ff_fill_uniform(C_panel, mr, cfg.n, cfg.n, cfg.p, cfg.seed, ffgen.STREAM_C, index0=r0 * cfg.n)
    in_bytes = 4 * (cfg.m * cfg.k + cfg.k * cfg.n)
    flush = in_bytes < 2 * L2_BYTES
    scratch = torch.empty(2 * L2_BYTES // 4, dtype=torch.int32, device=dev) if flush else None
    torch.cuda.synchronize()

    def barrier():
        if world > 1:
            if share:
                dist.barrier()
            else:
                dist.barrier(device_ids=[local])

    # ---- warm-up
    for _ in range(args.warmup):
        eng.step(A_panel, B, C_panel)
    torch.cuda.synchronize()
    barrier()
    torch.cuda.synchronize()

    # ---- timed region
    cur = torch.cuda.current_stream()
    gemm_ms, gemm_launches, launches = [], 0, 0
    with ClockSampler(local) as clk:
        if not flush:
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(cur)
            evs = []
            for _ in range(args.steps):
                eng.step(A_panel, B, C_panel, time_gemm=True)
                evs.append(list(eng.gemm_events))
                launches += eng.launches_per_step
            e1.record(cur)
            torch.cuda.synchronize()
            elapsed_ms = e0.elapsed_time(e1)
            for lst in evs:
                for a, b in lst:
                    gemm_ms.append(a.elapsed_time(b))
        else:
            elapsed_ms = 0.0
            for _ in range(args.steps):
                scratch.fill_(1)                     # L2 flush, untimed
                barrier()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(cur)
                eng.step(A_panel, B, C_panel, time_gemm=True)
                e1.record(cur)
                torch.cuda.synchronize()
                elapsed_ms += e0.elapsed_time(e1)
                gemm_ms += [a.elapsed_time(b) for a, b in eng.gemm_events]
                launches += eng.launches_per_step
    barrier()
    t = torch.tensor([elapsed_ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    elapsed_ms = float(t.item())
    gemm_launches = len(gemm_ms)
    ms_per_step = elapsed_ms / args.steps
    value = cfg.useful_ops() * args.steps / (elapsed_ms / 1e3) / 1e9      # GOPS, whole job

    # ---- roofline of the dominant kernel (the tcgen05 limb GEMM), this rank
    peaks = _peaks()
    chunk_units = [(b - a) for a, b in eng.chunks]
    ops_per_step = prods * 2.0 * mr * sum(chunk_units) * cfg.k          # int8 MMA ops (algorithmic)
    gemm_avg_ms = statistics.mean(gemm_ms) if gemm_ms else float("nan")
    ops_per_launch = ops_per_step / max(1, len(eng.chunks))
    achieved = ops_per_launch / (gemm_avg_ms / 1e3) / 1e12               # TOPS
    traffic = None
    prof = os.path.join(ROOT, "profiles", "ncu_gemm_%s.json" % cfg.name)
    if os.path.exists(prof):
        try:
            with open(prof) as f:
                pj = json.load(f)
            if pj.get("world", 1) == world:
                traffic = pj.get("dram_bytes_per_launch")
        except Exception:
            traffic = None
    roofline = {"bound": "tensor", "achieved": achieved, "peak": peaks["burst"], "unit": "TFLOP/s",
                "frac": achieved / peaks["burst"], "traffic": traffic,
                "kernel": "ffgemm_tc_kernel (tcgen05.mma.kind::i8)",
                "ops_per_launch": ops_per_launch, "ops_definition": "products (L^2 limb pairs, or n_q CRT moduli) * 2 * m_rank * n_chunk * k",
                "avg_launch_ms": gemm_avg_ms, "gemm_share_of_step": sum(gemm_ms) / elapsed_ms if elapsed_ms else None,
                "peak_source": peaks["source"] + ", burst figure (the timed region is well under a second)",
                "frac_of_sustained_peak": achieved / peaks["sustained"]}

    # ---- end to end through the public API with host buffers
    e2e = None
    if not args.no_e2e:
        e2e = run_e2e(args, cfg, eng, A_panel, B, C_panel, world, rank, local, dev)

    # ---- CPU baseline: the oracle on host cores (rank 0, N = 1 only)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        cpu, _ = cpu_oracle_sample(cfg)

    # clock-normalised tensor peak: 16384 int8 ops/clk/SM (one
    # 256x256x32 CTA-pair MMA per 128 cycles), at the median SM clock sampled
    # during the timed region
    clocks = clk.summary()
    try:
        nsm = torch.cuda.get_device_properties(dev).multi_processor_count
        if clocks.get("sm_mhz"):
            clk_peak = nsm * 16384 * clocks["sm_mhz"] * 1e6 / 1e12
            roofline["clock_peak"] = clk_peak
            roofline["frac_of_clock_peak"] = achieved / clk_peak
    except Exception:  # pragma: no cover - informational only
        pass
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "GOPS", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "int8",
            "data": "synthetic: seeded uniform residues in [0,p) (ffgen splitmix64 recipe), int32 in HBM",
            "config": _config_json(cfg, world, limbs=L, scheme=info["scheme"], kb=info["kb"],
                                   chunks=len(eng.chunks), l2=("flushed between steps (inputs < L2)" if flush
                                                               else "inputs larger than L2 (no flush)")),
            "tensor_pipe_pct": 100.0 * prods * cfg.useful_ops() * args.steps / (elapsed_ms / 1e3) / 1e12
            / (world * peaks["burst"]),
            "roofline": roofline,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": launches,
            "gemm_launches": gemm_launches,
            "clocks": clocks,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


def run_e2e(args, cfg, eng, A_panel, B, C_panel, world, rank, local, dev):
    """Same metric through the public API with pinned HOST buffers: each step
    copies the inputs host->device and the result device->host (timed)."""
    import ctypes
    import torch
    import torch.distributed as dist
    import paper_cs_0601133_b200 as ff

    mr = eng.mr
    hA = torch.empty(A_panel.shape, dtype=torch.int32, pin_memory=True)
    hA.copy_(A_panel)
    hB = None
    if rank == 0:
        hB = torch.empty(B.shape, dtype=torch.int32, pin_memory=True)
        hB.copy_(B)
    hC = torch.empty(C_panel.shape, dtype=torch.int32, pin_memory=True)
    hC.copy_(C_panel)
    beta_nz = cfg.beta % cfg.p != 0
    steps = max(1, min(args.steps, 5))
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
    a_bytes = 4 * cfg.m * cfg.k
    h2d = a_bytes + 4 * cfg.k * cfg.n + (4 * cfg.m * cfg.n if beta_nz else 0)
    d2h = 4 * cfg.m * cfg.n
    return {"value": cfg.useful_ops() * steps / (ms / 1e3) / 1e9, "unit": "GOPS", "steps": steps,
            "ms_per_step": ms / steps, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
            "api": "ff_gemm_host (C ABI, pinned host buffers)" if world == 1 else
            "RowPanelGemm.step with pinned host<->device copies per rank"}


if __name__ == "__main__":
    sys.exit(main())
