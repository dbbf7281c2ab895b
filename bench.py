#!/usr/bin/env python
"""Benchmark: fp64 recursive SPIKE factor + solve (+ transpose solve) on B200.

Default workload = BASELINE.json's metric config (configs[2], "C3"):
n=1,000,000, kl=ku=160, nrhs=160, dd=1.5, non-pivoting, one factorization
serving A X = F and A^T X = F.  One step = spk_factorize + spk_solve +
spk_solve(transpose) over the whole system; the metric is fp64 GFLOP/s of the
SPIKE-algorithmic work (factor 8nk^2, each solve 8nk*nrhs),
higher is better, with time per step beside it.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config c1..c5] [--impl ours|reference]

N > 1 (torchrun, one process per GPU, NCCL): strong scaling -- the
configuration's fixed system sharded into N slabs (--weak: N*n rows), each
GPU factoring and solving its slab with the slab-level reduced system
exchanged by all-gathers (paper_1811_03559_b200/distributed.py).

Inputs are seeded synthetic data (include/spike_b200_gen.h), generated in HBM
for the device-resident `value`, and in pinned host memory for `e2e`, which
goes through the public C-ABI with host buffers (copies inside the timed
region).  The CPU checkers/baselines under oracle/ are only used for the
`cpu_baseline` object (rank 0, N=1) and the `--impl reference` arm.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    "c1": dict(n=100_000, k=16, nrhs=1, dd=2.0, piv=False, transpose=False, bound="hbm",
               desc="C1 n=1e5 kl=ku=16 nrhs=1 dd=2.0 non-pivoting"),
    "c2": dict(n=1_000_000, k=64, nrhs=1, dd=1.1, piv=False, transpose=False, bound="fp64",
               desc="C2 n=1e6 kl=ku=64 nrhs=1 dd=1.1 non-pivoting"),
    "c3": dict(n=1_000_000, k=160, nrhs=160, dd=1.5, piv=False, transpose=True, bound="fp64",
               desc="C3 n=1e6 kl=ku=160 nrhs=160 dd=1.5 non-pivoting, solve + transpose solve"),
    "c4": dict(n=1_000_000, k=64, nrhs=4, dd=-1.0, piv=True, transpose=False, bound="fp64",
               desc="C4 n=1e6 kl=ku=64 nrhs=4 no dominance, partial pivoting"),
    "c5": dict(n=16_000_000, k=128, nrhs=32, dd=1.2, piv=False, transpose=False, bound="fp64",
               desc="C5 n=16e6 kl=ku=128 nrhs=32 dd=1.2 non-pivoting"),
}
SEED_A = 20181108
HBM_PEAK_FALLBACK = 6650.0
FP64_PEAK_MEASURED = 37.1  # TFLOP/s, tools/fp64_peak.cu on this pool's B200 (DMMA 37.1, DFMA 36.9)


def alg_flops(cfg):
    n, k, r = cfg["n"], cfg["k"], cfg["nrhs"]
    fac = (14.0 if cfg["piv"] else 8.0) * n * k * k
    sol = (12.0 if cfg["piv"] else 8.0) * n * k * r
    useful_fac = (4.0 if cfg["piv"] else 2.0) * n * k * k
    useful_sol = (6.0 if cfg["piv"] else 4.0) * n * k * r
    nsol = 2 if cfg["transpose"] else 1
    return fac + nsol * sol, useful_fac + nsol * useful_sol


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f)
    except Exception:
        return {}


class ClockSampler:
    """nvidia-smi clocks and throttle reasons sampled during the timed region."""

    def __init__(self, index=0):
        self.index = index
        self.samples = []
        self.proc = None

    def __enter__(self):
        q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "50"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [x.strip() for x in line.split(",")]
            if len(parts) >= 7:
                self.samples.append(parts)

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = sorted(float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit())
        mx = max((float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()), default=None)
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4) if s[3 + i].lower() == "active"})
        return {"sm_mhz": sm[len(sm) // 2] if sm else None, "sm_max_mhz": mx, "reasons": reasons,
                "samples": len(self.samples)}


# ----------------------------------------------------------------------------
# reference CPU arm (the compiled unmodified reference library, oracle/_ref)


def _ref_libs():
    from oracle.oracle import Oracle, Reference, build as obuild
    if not os.path.exists(os.path.join(ROOT, "oracle", "liboracle.so")):
        obuild(with_ref=False)
    ref = Reference.load()
    return Oracle(), ref


def host_cpu():
    """lscpu model, physical cores and logical CPUs of this host."""
    info = {"model": None, "physical_cores": None, "logical_cpus": os.cpu_count()}
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        kv = {}
        for line in out.splitlines():
            if ":" in line:
                a, b = line.split(":", 1)
                kv[a.strip()] = b.strip()
        info["model"] = kv.get("Model name")
        cps, sockets = kv.get("Core(s) per socket"), kv.get("Socket(s)")
        if cps and sockets and cps.isdigit() and sockets.isdigit():
            info["physical_cores"] = int(cps) * int(sockets)
    except Exception:
        pass
    return info


def reference_full(cfg, t, steps, want_x=False):
    """The reference CPU path (make_plan(t) -> factorize -> solve
    [-> transpose_solve], spike_cli.cpp:119-169) on the FULL configuration,
    `steps` times; returns the per-step seconds, p and (optionally) X / X^T of
    the last step."""
    o, ref = _ref_libs()
    k, nrhs, n = cfg["k"], cfg["nrhs"], cfg["n"]
    band = o.generate_band(SEED_A, n, k, k, cfg["dd"])
    F = o.generate_rhs(SEED_A + 1, n, nrhs)
    times, parts, p, X, XT = [], [], None, None, None
    for i in range(steps):
        r = ref.time_path(band, n, k, k, F, t, 1.0, cfg["piv"], cfg["transpose"], want_x=want_x and i == steps - 1)
        times.append(r["factor"] + r["solve"] + r["tsolve"])
        parts.append([r["factor"], r["solve"], r["tsolve"]])
        p = r["p"]
        if r["X"] is not None:
            X, XT = r["X"], r["XT"]
    return times, parts, p, X, XT


def reference_step_sample(cfg, target_s=8.0, t=None, calib=None):
    """Pick a row count so one reference factor+solve(s) step takes ~target_s."""
    o, ref = _ref_libs()
    t = t or os.cpu_count()
    k, nrhs = cfg["k"], cfg["nrhs"]
    n0 = calib or max(40 * (2 * k + 1) * 4, 20000)
    n0 = min(n0, cfg["n"])
    band = o.generate_band(SEED_A, n0, k, k, cfg["dd"])
    F = o.generate_rhs(SEED_A + 1, n0, nrhs)
    r = ref.time_path(band, n0, k, k, F, t, 1.0, cfg["piv"], cfg["transpose"])
    per_row = (r["factor"] + r["solve"] + r["tsolve"]) / n0
    n_s = int(min(cfg["n"], max(n0, target_s / max(per_row, 1e-12))))
    return n_s, t


def run_reference_steps(cfg, n_s, t, steps):
    o, ref = _ref_libs()
    k, nrhs = cfg["k"], cfg["nrhs"]
    band = o.generate_band(SEED_A, n_s, k, k, cfg["dd"])
    F = o.generate_rhs(SEED_A + 1, n_s, nrhs)
    times = []
    p = None
    for _ in range(steps):
        r = ref.time_path(band, n_s, k, k, F, t, 1.0, cfg["piv"], cfg["transpose"])
        times.append(r["factor"] + r["solve"] + r["tsolve"])
        p = r["p"]
    return times, p


def impl_reference(args, cfg):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    from oracle.oracle import Reference
    if Reference.load() is None:
        print(json.dumps({"impl": "reference", "unavailable":
                          "oracle/_ref/libspike_ref.so not built (reference sources absent at build time)"}))
        return 0
    hc = host_cpu()
    t = hc["physical_cores"] or os.cpu_count()
    # the full configuration (same n, k, nrhs, dd as our arm); C5 alone is
    # sampled when the whole run would exceed ~15 min on the host cores
    n_s = cfg["n"]
    if cfg["n"] > 4_000_000:
        n_est, _ = reference_step_sample(cfg, target_s=8.0, t=t)
        per_step = 8.0 * cfg["n"] / max(n_est, 1)
        if per_step * (args.steps + args.warmup) > 900.0:
            n_s = int(cfg["n"] * 900.0 / (per_step * (args.steps + args.warmup)))
    run_cfg = dict(cfg, n=n_s)
    times, parts, p, _, _ = reference_full(run_cfg, t, args.warmup + args.steps)
    timed = sorted(times[args.warmup:])
    fl, useful = alg_flops(run_cfg)
    ms = 1e3 * sum(timed) / len(timed)
    value = fl / (ms * 1e-3) / 1e9
    sample = (f"full system n={n_s}" if n_s == cfg["n"] else f"n={n_s} of {cfg['n']} rows (same k/nrhs/dd)") + \
        f"; reference make_plan(t={t}) -> p={p}; factorize+solve" + \
        ("+transpose_solve" if cfg["transpose"] else "") + f"; median step {timed[len(timed) // 2]:.3f} s"
    line = {"metric": args.metric, "value": round(value, 3), "unit": "GFLOP/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms, 3),
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded counter-based generator, include/spike_b200_gen.h)",
            "config": {"workload": cfg["desc"], "n": n_s, "kl": cfg["k"], "ku": cfg["k"], "nrhs": cfg["nrhs"],
                       "threads": t, "partitions": p, "host_cpu": hc,
                       "phase_seconds_median": [sorted(x[i] for x in parts[args.warmup:])[len(timed) // 2]
                                                for i in range(3)]},
            "impl": "reference",
            "cpu_baseline": {"value": round(value, 3), "unit": "GFLOP/s", "cores": t, "kind": "reference",
                             "sample": sample, "cpu_model": hc["model"]},
            "e2e": {"value": round(value, 3), "unit": "GFLOP/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line))
    return 0


# ----------------------------------------------------------------------------
# our arm


def band_norm(band, chunk=1 << 20):
    """max column abs-sum of the packed band (||A||_1) without a band-sized temporary."""
    m = 0.0
    for i in range(0, band.shape[0], chunk):
        m = max(m, band[i:i + chunk].abs().sum(dim=1).max().item())
    return m


def profile_roofline(spk, cfg, steps, ms):
    """Per-kernel-class device time inside the timed region -> roofline object
    for the dominant class."""
    import ctypes as C
    prof = {}
    ncls = spk.lib().spk_profile_classes()
    spk.lib().spk_profile_read.restype = C.c_char_p
    spk.lib().spk_profile_read.argtypes = [C.c_int32, C.POINTER(C.c_double), C.POINTER(C.c_double),
                                           C.POINTER(C.c_double), C.POINTER(C.c_int64)]
    for c in range(ncls):
        a, b, d, e = C.c_double(), C.c_double(), C.c_double(), C.c_int64()
        name = spk.lib().spk_profile_read(c, C.byref(a), C.byref(b), C.byref(d), C.byref(e)).decode()
        if e.value:
            prof[name] = dict(ms=a.value / steps, flops=b.value / steps, bytes=d.value / steps,
                              launches=e.value // steps)
    bound = cfg["bound"]
    # the dominant class; for HBM-bound configurations the dominant class that
    # moves algorithmic bytes (the small-k engine's level kernel moves k x k
    # tips only and is reported in `classes`)
    cand = {kk: v for kk, v in prof.items() if bound != "hbm" or v["bytes"] > 0} or prof
    top = max(cand.items(), key=lambda kv: kv[1]["ms"]) if cand else ("none", dict(ms=1, flops=0, bytes=0, launches=1))
    peaks = measured_peaks()
    tms = top[1]["ms"]
    if bound == "hbm":
        ach = top[1]["bytes"] / (tms * 1e-3) / 1e9
        peak = peaks.get("hbm_gbs", HBM_PEAK_FALLBACK)
        unit = "GB/s"
    else:
        ach = top[1]["flops"] / (tms * 1e-3) / 1e12
        peak = FP64_PEAK_MEASURED
        unit = "TFLOP/s"
    # DRAM bytes per launch of that kernel class from the committed ncu capture
    # (profiles/traffic.json), when one exists for this workload
    traffic = None
    try:
        tj = json.load(open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "profiles", "traffic.json")))
        ent = tj.get(cfg["desc"].split()[0], {}).get(top[0])
        if ent:
            traffic = (ent["bytes_per_launch"], ent["kernel"] + "; " + ent["source"])
    except (OSError, ValueError):
        pass
    return {"bound": bound, "kernel": top[0], "achieved": round(ach, 3), "peak": peak, "unit": unit,
            "frac": round(ach / peak, 4), "traffic": traffic[0] if traffic else None,
            "traffic_unit": "bytes per launch (dram read + write)", "traffic_source": traffic[1] if traffic else None,
            "kernel_share_of_step": round(tms / ms, 4),
            "peak_source": ("MEASURED_PEAKS.json hbm_gbs" if bound == "hbm"
                            else "tools/fp64_peak.cu measured DMMA/DFMA peak on this pool (B200)"),
            "classes": {kk: {"ms": round(v["ms"], 4), "launches": v["launches"]} for kk, v in prof.items()}}


def impl_ours_slabs(args, cfg, spk, torch, dist, rank, world, dev):
    """N > 1 (or --slabs): the configuration's system sharded into N slabs
    (strong scaling; --weak: N*n rows), each GPU factoring its slab through the
    C++ data plane (csrc/spk_dist.cu); the only collectives are the library's
    NCCL all-gathers of the slab-level reduced system's tip blocks."""
    from paper_1811_03559_b200 import distributed as D
    stream = torch.cuda.current_stream(dev)
    sptr = stream.cuda_stream
    lib = spk.lib()
    k, nrhs = cfg["k"], cfg["nrhs"]
    # strong scaling (default): the configuration's fixed system sharded over
    # the GPUs, as BASELINE C5 specifies; --weak: n rows per GPU
    n_glob = world * cfg["n"] if args.weak else cfg["n"]
    n_loc = n_glob // world
    rows = D.slab_rows(n_glob, world)
    r0, r1 = rows[rank], rows[rank + 1]
    n = r1 - r0
    lh, rh = D.halo(rank, world, k)
    ld = 2 * k + 1
    band = torch.empty((n + lh + rh, ld), dtype=torch.float64, device=dev)  # slab + halo columns
    F = torch.empty((nrhs, n), dtype=torch.float64, device=dev)
    X = torch.empty_like(F)
    XT = torch.empty_like(F)
    spk.spike._check(lib.spk_generate_band_cols(SEED_A, n_glob, k, k, cfg["dd"], r0 - lh, n + lh + rh,
                                                 band.data_ptr(), sptr))
    spk.spike._check(lib.spk_generate_rhs_rows(SEED_A + 1, r0, n, nrhs, F.data_ptr(), n, sptr))
    plan = spk.gpu_plan(n, k, k, nrhs, cfg["piv"], args.p)
    opts = spk.FactorOptions(pivoting=cfg["piv"])
    # the C++ data plane (csrc/spk_dist.cu): the library's own NCCL
    # communicator (unique id broadcast over the process group); it issues the
    # tip all-gathers itself on this stream
    plane = D.NcclPlane()

    def run_step(band_t, F_t, X_t, XT_t):
        df = plane.factorize(band_t.data_ptr(), n, k, k, plan, opts, sptr)
        plane.solve(df, F_t.data_ptr(), n, nrhs, X_t.data_ptr(), n, False, sptr)
        if cfg["transpose"]:
            plane.solve(df, F_t.data_ptr(), n, nrhs, XT_t.data_ptr(), n, True, sptr)

    def step():
        run_step(band, F, X, XT)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    # correctness guard: backward error of this slab's rows of A X = F, with the
    # neighbours' edge rows of X gathered into the halo
    step()
    edge = torch.cat([X[:, :k], X[:, n - k:]], dim=1).contiguous()
    parts = [torch.empty_like(edge) for _ in range(world)]
    dist.all_gather(parts, edge)
    Xe = torch.zeros((nrhs, n + lh + rh), dtype=torch.float64, device=dev)
    Xe[:, lh:lh + n] = X
    if lh:
        Xe[:, :k] = parts[rank - 1][:, k:]
    if rh:
        Xe[:, lh + n:] = parts[rank + 1][:, :k]
    R = torch.empty_like(Xe)
    lib.spk_band_matmul(band.data_ptr(), n + lh + rh, k, k, Xe.data_ptr(), n + lh + rh, nrhs, 0, R.data_ptr(),
                        n + lh + rh, 1, sptr)
    anorm = band_norm(band)
    berr_t = ((R[:, lh:lh + n] - F).abs().amax(dim=1) / (anorm * X.abs().amax(dim=1))).max().reshape(1)
    dist.all_reduce(berr_t, op=dist.ReduceOp.MAX)
    berr = berr_t.item()
    del R, Xe
    torch.cuda.empty_cache()  # the library's own arena allocates next

    dist.barrier()
    torch.cuda.synchronize()
    lib.spk_launch_count(1)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    with ClockSampler(int(os.environ.get("LOCAL_RANK", "0"))) as clk:
        for i in range(args.steps):
            ev[i][0].record(stream)
            step()
            ev[i][1].record(stream)
        torch.cuda.synchronize()
    launches = int(lib.spk_launch_count(1))
    ms_t = torch.tensor([sum(a.elapsed_time(b) for a, b in ev) / args.steps], device=dev)
    dist.all_reduce(ms_t, op=dist.ReduceOp.MAX)
    ms = ms_t.item()
    fl, useful = alg_flops(dict(cfg, n=n_glob))
    value = fl / (ms * 1e-3) / 1e9
    lib.spk_profile_reset()
    lib.spk_profile_enable(1)
    step()
    torch.cuda.synchronize()
    lib.spk_profile_enable(0)
    roofline = profile_roofline(spk, cfg, 1, ms)

    e2e = None
    if not args.no_e2e:
        hband = band.cpu().pin_memory()
        hF = F.cpu().pin_memory()
        hX = torch.empty_like(hF).pin_memory()
        hXT = torch.empty_like(hF).pin_memory()
        del band, F, X, XT, step  # the e2e leg stages its own device copies
        torch.cuda.empty_cache()
        lib.spk_arena_trim()
        dband = torch.empty(hband.shape, dtype=torch.float64, device=dev)
        dF, dX, dXT = (torch.empty(hF.shape, dtype=torch.float64, device=dev) for _ in range(3))

        def e2e_step():
            dband.copy_(hband, non_blocking=True)
            dF.copy_(hF, non_blocking=True)
            run_step(dband, dF, dX, dXT)
            hX.copy_(dX, non_blocking=True)
            if cfg["transpose"]:
                hXT.copy_(dXT, non_blocking=True)

        e2e_step()
        torch.cuda.synchronize()
        dist.barrier()
        e_steps = max(1, min(args.steps, 5))
        t0 = time.perf_counter()
        for _ in range(e_steps):
            e2e_step()
        torch.cuda.synchronize()
        ems_t = torch.tensor([(time.perf_counter() - t0) * 1e3 / e_steps], device=dev)
        dist.all_reduce(ems_t, op=dist.ReduceOp.MAX)
        ems = ems_t.item()
        nsol = 2 if cfg["transpose"] else 1
        e2e = {"value": round(fl / (ems * 1e-3) / 1e9, 3), "unit": "GFLOP/s", "ms_per_step": round(ems, 3),
               "h2d_bytes_per_step": int(world * (hband.numel() + hF.numel()) * 8),
               "d2h_bytes_per_step": int(world * nsol * hX.numel() * 8)}

    if rank == 0:
        line = {"metric": args.metric, "value": round(value, 3), "unit": "GFLOP/s", "n_gpus": world,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms, 4),
                "higher_is_better": True, "scaling": "weak" if args.weak else "strong", "vs_baseline": None,
                "dtype": "f64",
                "data": "synthetic (seeded counter-based generator, include/spike_b200_gen.h; each GPU "
                        "generates its slab + halo columns in HBM)",
                "config": {"workload": cfg["desc"] + (f"; weak scaling: one global system of {world} x n rows"
                                                      if args.weak else f"; strong scaling over {world} GPUs"),
                           "n": n_glob, "n_per_gpu": n_loc, "kl": k, "ku": k, "nrhs": nrhs,
                           "partitions_per_gpu": plan.p,
                           "parallelism": f"slabs{world} (NCCL tip all-gathers issued by the C++ data plane)",
                           "l2": "inputs larger than L2"},
                "useful_gflops": round(useful / (ms * 1e-3) / 1e9, 3),
                "backward_error": berr,
                "roofline": roofline, "cpu_baseline": None, "e2e": e2e, "gpu_launches": launches,
                "clocks": clk.summary(), "impl": "ours"}
        print(json.dumps(line))
    dist.destroy_process_group()
    return 0


def small_k_leg(spk, torch, dev, stream, steps=10, warmup=3):
    """The BASELINE metric's "HBM GB/s small-k" half: C1 (n=1e5, kl=ku=16,
    nrhs=1) factor + solve on the device, L2 flushed between steps; bytes are
    SURVEY 8(d)'s algorithmic counts (factor: read A + write factors, solve: two
    factor reads + F in, Y, X)."""
    c = CONFIGS["c1"]
    n, k, nrhs = c["n"], c["k"], c["nrhs"]
    sptr = stream.cuda_stream
    band = torch.empty((n, 2 * k + 1), dtype=torch.float64, device=dev)
    F = torch.empty((nrhs, n), dtype=torch.float64, device=dev)
    X = torch.empty_like(F)
    spk.generate_band_device(SEED_A, n, k, k, c["dd"], band.data_ptr(), sptr)
    spk.generate_rhs_device(SEED_A + 1, n, nrhs, F.data_ptr(), n, sptr)
    plan = spk.gpu_plan(n, k, k, nrhs, False, 0)
    opts = spk.FactorOptions(pivoting=False)
    flush = torch.empty(64 * 2 ** 20, dtype=torch.float64, device=dev)
    # the C-ABI calls themselves (spk_factorize, spk_solve, spk_fact_destroy):
    # stream-ordered, no host wait inside a step (the small-k engine needs no
    # host-side finish before its solve)
    import ctypes as C
    L = spk.lib()
    st, keep = spk.spike._plan_struct(plan)
    o = spk.spike._Opts(0, opts.boost_eps)

    def step():
        h = C.c_void_p()
        spk.spike._check(L.spk_factorize(C.c_void_p(band.data_ptr()), 1, n, k, k, C.byref(st), C.byref(o), sptr,
                                          C.byref(h)))
        spk.spike._check(L.spk_solve(h, 0, C.c_void_p(F.data_ptr()), n, nrhs, C.c_void_p(X.data_ptr()), n, 1,
                                     sptr, None))
        L.spk_fact_destroy(h)

    for _ in range(warmup):
        step()
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
    for i in range(steps):
        flush.zero_()
        ev[i][0].record(stream)
        step()
        ev[i][1].record(stream)
    torch.cuda.synchronize()
    ms = sum(a.elapsed_time(b) for a, b in ev) / steps
    fbytes = 16.0 * n * (2 * k + 1)
    sbytes = 2 * 8.0 * n * (2 * k + 1) + 32.0 * n * nrhs
    gbs = (fbytes + sbytes) / (ms * 1e-3) / 1e9
    peak = measured_peaks().get("hbm_gbs", HBM_PEAK_FALLBACK)
    del band, F, X, flush
    return {"workload": c["desc"], "ms_per_step": round(ms, 4), "hbm_gbs": round(gbs, 2),
            "bytes_per_step": int(fbytes + sbytes), "peak_gbs": peak, "frac": round(gbs / peak, 5),
            "partitions": plan.p, "engine": "small-k (3 launches per step: k_sk_parts, k_sk_levels, k_sk_solve)"}


def impl_ours(args, cfg):
    import torch
    import torch.distributed as dist
    import paper_1811_03559_b200 as spk
    from paper_1811_03559_b200 import build as pbuild
    if not os.path.exists(spk.LIB_PATH):
        pbuild.build()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1 or args.slabs:
        dist.init_process_group("nccl", device_id=dev)
        return impl_ours_slabs(args, cfg, spk, torch, dist, rank, world, dev)
    stream = torch.cuda.current_stream(dev)
    sptr = stream.cuda_stream

    n, k, nrhs = cfg["n"], cfg["k"], cfg["nrhs"]
    ld = 2 * k + 1
    band = torch.empty((n, ld), dtype=torch.float64, device=dev)
    F = torch.empty((nrhs, n), dtype=torch.float64, device=dev)   # column-major n x nrhs
    X = torch.empty_like(F)
    XT = torch.empty_like(F)
    spk.generate_band_device(SEED_A, n, k, k, cfg["dd"], band.data_ptr(), sptr)
    spk.generate_rhs_device(SEED_A + 1, n, nrhs, F.data_ptr(), n, sptr)
    plan = spk.gpu_plan(n, k, k, nrhs, cfg["piv"], args.p)
    opts = spk.FactorOptions(pivoting=cfg["piv"])
    L2_BYTES = 126 * 2 ** 20
    flush = None
    if band.numel() * 8 < 2 * L2_BYTES:
        flush = torch.empty(64 * 2 ** 20, dtype=torch.float64, device=dev)  # 512 MB

    def step():
        fact = spk.factorize_device(band.data_ptr(), n, k, k, plan, opts, sptr)
        spk.solve_device(fact, F.data_ptr(), n, nrhs, X.data_ptr(), n, False, sptr)
        if cfg["transpose"]:
            spk.solve_device(fact, F.data_ptr(), n, nrhs, XT.data_ptr(), n, True, sptr)
        return fact

    # the timed step: the C-ABI calls themselves (spk_factorize, spk_solve,
    # spk_fact_destroy), stream-ordered; the library host-syncs only where its
    # programs need the factorization's outcome (the general engine's finish)
    import ctypes as C
    L = spk.lib()
    cst, ckeep = spk.spike._plan_struct(plan)
    copt = spk.spike._Opts(int(cfg["piv"]), opts.boost_eps)

    def timed_step():
        h = C.c_void_p()
        spk.spike._check(L.spk_factorize(C.c_void_p(band.data_ptr()), 1, n, k, k, C.byref(cst), C.byref(copt), sptr,
                                          C.byref(h)))
        spk.spike._check(L.spk_solve(h, 0, C.c_void_p(F.data_ptr()), n, nrhs, C.c_void_p(X.data_ptr()), n, 1,
                                     sptr, None))
        if cfg["transpose"]:
            spk.spike._check(L.spk_solve(h, 1, C.c_void_p(F.data_ptr()), n, nrhs, C.c_void_p(XT.data_ptr()), n, 1,
                                         sptr, None))
        L.spk_fact_destroy(h)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    # correctness guard on the benchmarked system: normwise backward error on device
    fact = step()
    lib = spk.lib()
    # max_c ||f_c - op(A) x_c||_inf / (||op(A)||_inf ||x_c||_inf), residual on the tensor cores
    berr = spk.backward_error_device(band.data_ptr(), n, k, k, X.data_ptr(), n, F.data_ptr(), n, nrhs, False, sptr)
    if cfg["transpose"]:
        berr = max(berr, spk.backward_error_device(band.data_ptr(), n, k, k, XT.data_ptr(), n, F.data_ptr(), n,
                                                   nrhs, True, sptr))
    del fact
    # host copies of the device solutions: compared with the reference's
    # (cpu_baseline leg) and with the e2e leg's host-buffer results
    hXdev = X.cpu()
    hXTdev = XT.cpu() if cfg["transpose"] else None
    torch.cuda.empty_cache()  # the library's own arena allocates next

    torch.cuda.synchronize()
    spk.lib().spk_launch_count(1)
    spk.lib().spk_generic_launch_count(1)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    for _ in range(2):
        timed_step()
    torch.cuda.synchronize()
    spk.lib().spk_launch_count(1)
    spk.lib().spk_generic_launch_count(1)
    with ClockSampler(local) as clk:
        for i in range(args.steps):
            if flush is not None:
                flush.zero_()
            ev[i][0].record(stream)
            timed_step()
            ev[i][1].record(stream)
        torch.cuda.synchronize()
    launches = int(spk.lib().spk_launch_count(1))
    generic = int(spk.lib().spk_generic_launch_count(1))
    ms = sum(a.elapsed_time(b) for a, b in ev) / args.steps
    fl, useful = alg_flops(cfg)
    value = fl / (ms * 1e-3) / 1e9

    # per-kernel-class device time from separate profiled steps (the per-launch
    # events would inflate the timed ones)
    spk.lib().spk_profile_reset()
    spk.lib().spk_profile_enable(1)
    nprof = 2
    for _ in range(nprof):
        if flush is not None:
            flush.zero_()
        step()
    torch.cuda.synchronize()
    spk.lib().spk_profile_enable(0)
    roofline = profile_roofline(spk, cfg, nprof, ms)
    l2_note = "inputs larger than L2" if flush is None else "L2 flushed between steps"

    # configurations whose step has no transposed solve: one A^T X = F from the
    # step's factorization, reported beside the step (north_star: transpose
    # solves for both variants; C4's is the pivoted transposed path)
    tr_info = None
    if not cfg["transpose"]:
        fact = spk.factorize_device(band.data_ptr(), n, k, k, plan, opts, sptr)
        spk.solve_device(fact, F.data_ptr(), n, nrhs, XT.data_ptr(), n, True, sptr)  # (row-major copy made here)
        torch.cuda.synchronize()
        tev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(3)]
        for a_, b_ in tev:
            if flush is not None:
                flush.zero_()
            a_.record(stream)
            spk.solve_device(fact, F.data_ptr(), n, nrhs, XT.data_ptr(), n, True, sptr)
            b_.record(stream)
        torch.cuda.synchronize()
        tms = sum(a_.elapsed_time(b_) for a_, b_ in tev) / len(tev)
        tberr = spk.backward_error_device(band.data_ptr(), n, k, k, XT.data_ptr(), n, F.data_ptr(), n, nrhs, True,
                                          sptr)
        tr_info = {"ms": round(tms, 4), "gflops": round((12.0 if cfg["piv"] else 8.0) * n * k * nrhs /
                                                        (tms * 1e-3) / 1e9, 3),
                   "backward_error": tberr,
                   "note": "one transposed solve from the step's factorization (not part of the timed step)"}
        del fact

    # e2e through the public C-ABI with pinned host buffers
    e2e = None
    if not args.no_e2e:
        hband = band.cpu().pin_memory()
        hF = F.cpu().pin_memory()
        hX = torch.empty_like(hF).pin_memory()
        hXT = torch.empty_like(hF).pin_memory()
        # the e2e leg stages its own device copies: release the resident inputs
        del band, F, X, XT, flush, step
        torch.cuda.empty_cache()
        lib.spk_arena_trim()

        def e2e_step():
            fct = spk.lib()
            h = spk.spike.C.c_void_p()
            st, keep = spk.spike._plan_struct(plan)
            o = spk.spike._Opts(int(cfg["piv"]), opts.boost_eps)
            spk.spike._check(fct.spk_factorize(hband.data_ptr(), 0, n, k, k, spk.spike.C.byref(st),
                                               spk.spike.C.byref(o), sptr, spk.spike.C.byref(h)))
            spk.spike._check(fct.spk_solve(h, 0, hF.data_ptr(), n, nrhs, hX.data_ptr(), n, 0, sptr, None))
            if cfg["transpose"]:
                spk.spike._check(fct.spk_solve(h, 1, hF.data_ptr(), n, nrhs, hXT.data_ptr(), n, 0, sptr, None))
            fct.spk_fact_destroy(h)
            # host X / X^T complete (stream-ordered host solves): no overlap across steps
            spk.spike._check(fct.spk_stream_sync(sptr))

        e2e_step()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        e_steps = max(1, min(args.steps, 5))
        for _ in range(e_steps):
            e2e_step()
        torch.cuda.synchronize()
        ems = (time.perf_counter() - t0) * 1e3 / e_steps
        nsol = 2 if cfg["transpose"] else 1
        same = bool(torch.equal(hX, hXdev)) and (not cfg["transpose"] or bool(torch.equal(hXT, hXTdev)))
        e2e = {"value": round(fl / (ems * 1e-3) / 1e9, 3), "unit": "GFLOP/s",
               "ms_per_step": round(ems, 3),
               "h2d_bytes_per_step": int(hband.numel() * 8 + nsol * hF.numel() * 8),
               "d2h_bytes_per_step": int(nsol * hX.numel() * 8),
               "x_bit_identical_to_device_run": same}

    # CPU baseline: the compiled reference on the box's host cores (rank 0, N=1)
    # the full system (C5: a row sample, its host RAM and ~1 min per step), median
    # of 3 steps on all physical cores (spike_cli.cpp:80-91), plus a t=1 figure
    # on a bounded row sample; the reference's X / X^T of the full run are
    # compared with the GPU's
    cpu = None
    if not args.no_cpu:
        try:
            from oracle.oracle import Reference
            if Reference.load() is not None:
                hc = host_cpu()
                t = hc["physical_cores"] or os.cpu_count()
                n_s = n if n <= 4_000_000 else 1_000_000
                times, parts, p, Xr, XTr = reference_full(dict(cfg, n=n_s), t, 3, want_x=(n_s == n))
                med = sorted(times)[1]
                fls, _ = alg_flops(dict(cfg, n=n_s))
                n1, t1 = reference_step_sample(cfg, target_s=4.0, t=1)
                fl1, _ = alg_flops(dict(cfg, n=n1))
                t1s, _ = run_reference_steps(cfg, n1, 1, 1)
                cpu = {"value": round(fls / med / 1e9, 3), "unit": "GFLOP/s", "cores": t, "kind": "reference",
                       "cpu_model": hc["model"], "logical_cpus": hc["logical_cpus"],
                       "sample": (f"full system n={n}" if n_s == n else f"n={n_s} of {n} rows (same k/nrhs/dd)") +
                                 f", reference make_plan(t={t}) -> p={p}, median of 3 factorize+solve" +
                                 ("+transpose_solve" if cfg["transpose"] else "") +
                                 f" steps: {med:.3f} s (all: " + ", ".join(f"{x:.3f}" for x in times) + ")",
                       "phase_seconds_median": [sorted(x[i] for x in parts)[1] for i in range(3)],
                       "t1": {"value": round(fl1 / t1s[0] / 1e9, 3), "unit": "GFLOP/s", "cores": 1,
                              "sample": f"n={n1} rows, make_plan(t=1), one step in {t1s[0]:.2f} s"}}
                if Xr is not None:
                    xr = torch.from_numpy(np.ascontiguousarray(Xr.T))
                    cpu["dx_vs_gpu"] = (hXdev - xr).abs().max().item() / xr.abs().max().item()
                    if cfg["transpose"] and XTr is not None:
                        xtr = torch.from_numpy(np.ascontiguousarray(XTr.T))
                        cpu["dx_vs_gpu_transpose"] = (hXTdev - xtr).abs().max().item() / xtr.abs().max().item()
        except Exception as ex:  # pragma: no cover
            cpu = {"value": None, "error": str(ex)[:200]}

    small = None
    if args.config == "c3" and not args.no_small_k:
        torch.cuda.empty_cache()
        small = small_k_leg(spk, torch, dev, stream)

    if rank == 0:
        line = {"metric": args.metric, "value": round(value, 3), "unit": "GFLOP/s", "n_gpus": 1,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms, 4),
                "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
                "data": "synthetic (seeded counter-based generator, include/spike_b200_gen.h; generated in HBM)",
                "config": {"workload": cfg["desc"], "n": n, "kl": k, "ku": k, "nrhs": nrhs,
                           "partitions": plan.p, "parallelism": "1gpu",
                           "l2": l2_note},
                "useful_gflops": round(useful / (ms * 1e-3) / 1e9, 3),
                "backward_error": berr,
                "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches,
                "generic_kernel_launches": generic,
                "clocks": clk.summary(), "impl": "ours"}
        if small is not None:
            line["small_k"] = small
        if tr_info is not None:
            line["transpose_solve"] = tr_info
        print(json.dumps(line))
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="c3", choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--p", type=int, default=0, help="force the partition count")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-small-k", action="store_true", help="skip the C1 small-k HBM leg of the default line")
    ap.add_argument("--weak", action="store_true",
                    help="N > 1: n rows per GPU (one global system of N*n rows) instead of the fixed system")
    ap.add_argument("--slabs", action="store_true",
                    help="multi-GPU slab path even at N=1 (under torchrun; N>1 always uses it)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3) if args.impl == "ours" else args.warmup
    args.metric = "fp64 factor+solve GFLOP/s (SPIKE-algorithmic flops), " + CONFIGS[args.config]["desc"]
    cfg = CONFIGS[args.config]
    if args.impl == "reference":
        return impl_reference(args, cfg)
    return impl_ours(args, cfg)


if __name__ == "__main__":
    sys.exit(main())
