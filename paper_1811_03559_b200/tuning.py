"""Partition-ratio tuning on the GPU (the reference CLI's `calibrate` and
`sweep-ratios`, tools/spike_cli.cpp:171-227, partition.cpp:120-170).

`sweep_ratios` times the device-resident factorization and solve over a grid
of first/last-to-inner partition size ratios (the reference's R13; R12 has no
GPU counterpart because dual partitions factor like single ones) and adds the
point the calibrated K predicts (compute_ratios), flagged "calculated", with
the same CSV columns and gain line as the reference tool.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import List, Optional, Sequence

import torch

from . import spike as _spk


@dataclass
class RatioPoint:
    r12: float
    r13: float
    factor_seconds: float
    solve_seconds: float
    calculated: bool = False

    @property
    def total_seconds(self) -> float:
        return self.factor_seconds + self.solve_seconds


def _median_seconds(reps: int, fn, stream) -> float:
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        fn()
        b.record(stream)
        b.synchronize()
        ts.append(a.elapsed_time(b) * 1e-3)
    ts.sort()
    return ts[len(ts) // 2]


def sweep_ratios(n: int, k: int, nrhs: int, r13_values: Sequence[float], dd: float = 1.5, pivoting: bool = False,
                 p: int = 0, seed: int = 20181108, reps: int = 3, K: Optional[float] = None) -> List[RatioPoint]:
    """Times factor and solve (medians of `reps`, CUDA events) for each r13 and
    for the compute_ratios(K, nrhs, k) point (K from the cache or calibrate_k
    when not given)."""
    dev = torch.device("cuda", torch.cuda.current_device())
    stream = torch.cuda.current_stream(dev)
    sp = stream.cuda_stream
    band = torch.empty((n, 2 * k + 1), dtype=torch.float64, device=dev)
    F = torch.empty((nrhs, n), dtype=torch.float64, device=dev)
    X = torch.empty_like(F)
    _spk.generate_band_device(seed, n, k, k, dd, band.data_ptr(), sp)
    _spk.generate_rhs_device(seed + 1, n, nrhs, F.data_ptr(), n, sp)
    opts = _spk.FactorOptions(pivoting=pivoting)
    if K is None:
        K = _spk.read_k_cache(_spk.default_k_cache_path())
        if K is None:
            K = _spk.calibrate_k(0, k, 5).k
    c12, c13 = _spk.compute_ratios(K, nrhs, k)
    grid: List[RatioPoint] = []

    def run_point(r13: float, r12: float, calc: bool):
        plan = _spk.gpu_plan(n, k, k, nrhs, pivoting, p, r13=r13)
        holder = {}

        def fac():
            holder["f"] = _spk.factorize_device(band.data_ptr(), n, k, k, plan, opts, sp)

        fac()
        tf = _median_seconds(reps, fac, stream)
        fact = holder["f"]

        def sol():
            _spk.solve_device(fact, F.data_ptr(), n, nrhs, X.data_ptr(), n, False, sp)

        sol()
        ts = _median_seconds(reps, sol, stream)
        grid.append(RatioPoint(r12, r13, tf, ts, calc))

    for r13 in r13_values:
        run_point(float(r13), 1.0, False)
    run_point(float(c13), float(c12), True)
    return grid


def format_csv(grid: Sequence[RatioPoint]) -> str:
    """The reference tool's output: rows, then the gain of the calculated
    point over the best measured one (spike_cli.cpp:198-225)."""
    lines = ["r12,r13,factor_seconds,solve_seconds,total_seconds,flag"]
    for g in grid:
        lines.append(f"{g.r12:.4g},{g.r13:.4g},{g.factor_seconds:.6g},{g.solve_seconds:.6g},"
                     f"{g.total_seconds:.6g},{'calculated' if g.calculated else ''}")
    calc = grid[-1]
    bf = min(g.factor_seconds for g in grid)
    bs = min(g.solve_seconds for g in grid)
    bt = min(g.total_seconds for g in grid)
    lines.append(f"# gain_from_best_measured: factor={100 * abs(calc.factor_seconds / bf - 1):.2f}% "
                 f"solve={100 * abs(calc.solve_seconds / bs - 1):.2f}% "
                 f"combined={100 * abs(calc.total_seconds / bt - 1):.2f}%")
    return "\n".join(lines) + "\n"
