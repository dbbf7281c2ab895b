"""Randomised parity sweep: the GPU path against the CPU oracle's direct banded
solve over random shapes (asymmetric and one-sided bands, ragged nrhs, odd
partition counts, both factorization variants, forward and transpose, device
and host buffers, the former with padded leading dimensions).  Prints one JSON line per failure and a summary line.

  python tools/fuzz_parity.py [--cases N] [--seed S] [--seconds T]
"""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import paper_1811_03559_b200 as spk  # noqa: E402
from oracle.oracle import Oracle  # noqa: E402  (the checker)

RES_TOL, GAP_TOL = 1e-12, 1e-10


def rel_componentwise(x, y):
    return float(np.max(np.abs(x - y) / np.maximum(1.0, np.abs(y)))) if x.size else 0.0


def draw(rng):
    cls = rng.choice(["tiny", "small", "mid", "wide", "huge"], p=[0.2, 0.25, 0.25, 0.2, 0.1])
    kmax = {"tiny": 3, "small": 16, "mid": 64, "wide": 160, "huge": 200}[cls]
    kmin = {"tiny": 0, "small": 1, "mid": 17, "wide": 65, "huge": 161}[cls]
    k = int(rng.integers(kmin, kmax + 1))
    shape = rng.choice(["sym", "asym", "lower", "upper"], p=[0.5, 0.3, 0.1, 0.1])
    if shape == "sym":
        kl = ku = k
    elif shape == "asym":
        kl, ku = k, int(rng.integers(0, k + 1))
        if rng.random() < 0.5:
            kl, ku = ku, kl
    elif shape == "lower":
        kl, ku = k, 0
    else:
        kl, ku = 0, k
    kk = max(kl, ku, 1)
    p = int(rng.choice([1, 2, 3, 4, 5, 6, 7, 9, 12, 16, 23, 37]))
    per = int(rng.integers(2 * kk + 1, 6 * kk + 40))
    n = max(p * per + int(rng.integers(0, p + 1)), kl + ku + 2)
    if n > 60000:
        p = max(1, 60000 // per)
        n = p * per
    nrhs = int(rng.choice([1, 2, 3, 5, 8, 16, 31, 32, 33, 40, 64, 80, 81, 100, 160, 170]))
    if n * nrhs > 4_000_000:
        nrhs = max(1, 4_000_000 // n)
    piv = bool(rng.random() < 0.4)
    dd = float(rng.choice([1.2, 1.5, 2.0]))  # dominant: the direct solve is the bar (non-dominant
    # bands need the same-plan SPIKE oracle: tests/test_gpu_parity.py PIV_CASES)
    planner = rng.choice(["gpu", "ref"], p=[0.7, 0.3])
    c = dict(n=n, kl=kl, ku=ku, nrhs=nrhs, p=p, piv=piv, dd=dd, planner=str(planner),
             seed=int(rng.integers(1, 2**31 - 2)))
    # (drawn last: the shapes of a seed stay what they were before this option existed)
    c["device"] = bool(rng.random() < 0.5)
    c["padf"], c["padx"] = int(rng.choice([0, 1, 5, 64])), int(rng.choice([0, 3, 8]))
    return c


def run_case(o, c):
    n, kl, ku, nrhs = c["n"], c["kl"], c["ku"], c["nrhs"]
    band = o.generate_band(c["seed"], n, kl, ku, c["dd"])
    # the generator's diagonal is dd x the row's off-diagonal sum: a one-sided
    # band has an empty first or last row (exactly singular); give it a pivot
    band[band[:, ku] == 0.0, ku] = 1.5
    F = np.asfortranarray(o.generate_rhs(c["seed"] + 1, n, nrhs))
    a = spk.BandedMatrix(n, kl, ku, band)
    if c["planner"] == "gpu":
        plan = spk.gpu_plan(n, kl, ku, nrhs, c["piv"], c["p"])
    else:
        r12, r13 = spk.compute_ratios(1.0, nrhs, max(kl, ku, 1))
        plan = spk.make_plan(n, kl, ku, c["p"], r12, r13)
    c["p_used"] = plan.p
    dev = c.get("device", False)
    if dev:
        # device-resident band, F and X with padded leading dimensions (NaN in
        # the padding rows: they must be neither read into the result nor written)
        import torch
        s = torch.cuda.current_stream().cuda_stream
        dband = torch.from_numpy(np.ascontiguousarray(band)).cuda()
        ldf, ldx = n + c["padf"], n + c["padx"]
        dF = torch.full((nrhs, ldf), float("nan"), dtype=torch.float64, device="cuda")
        dF[:, :n] = torch.from_numpy(np.ascontiguousarray(F.T)).cuda()
        dX = torch.full((nrhs, ldx), float("nan"), dtype=torch.float64, device="cuda")
        fact = spk.factorize_device(dband.data_ptr(), n, kl, ku, plan, spk.FactorOptions(pivoting=c["piv"]), s)
    else:
        fact = spk.factorize(a, plan, spk.FactorOptions(pivoting=c["piv"]))
    out = {}
    for tr in (False, True):
        xo = o.oracle_solve(band, n, kl, ku, F, tr, True)  # pivoted direct banded solve
        if dev:
            dX.fill_(float("nan"))
            spk.solve_device(fact, dF.data_ptr(), ldf, nrhs, dX.data_ptr(), ldx, tr, s)
            torch.cuda.synchronize()
            if c["padx"] and not bool(torch.isnan(dX[:, n:]).all()):
                raise AssertionError("solve wrote X's padding rows")
            if not bool(torch.equal(dF[:, :n].cpu(), torch.from_numpy(np.ascontiguousarray(F.T)))):
                raise AssertionError("solve modified F")
            X = np.asfortranarray(dX[:, :n].cpu().numpy().T)
        else:
            X = spk.transpose_solve(fact, F) if tr else spk.solve(fact, F)
        res = o.relative_residual(band, n, kl, ku, X, F, tr)
        gap = rel_componentwise(X, xo)
        ores = o.relative_residual(band, n, kl, ku, xo, F, tr)
        out["T" if tr else "N"] = (res, gap, ores)
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cases", type=int, default=400)
    ap.add_argument("--seed", type=int, default=20181108)
    ap.add_argument("--seconds", type=float, default=600.0)
    a = ap.parse_args()
    o = Oracle(os.path.join(ROOT, "oracle", "liboracle.so"))
    rng = np.random.default_rng(a.seed)
    t0 = time.time()
    done = fails = rejected = 0
    worst_res = worst_gap = 0.0
    for i in range(a.cases):
        if time.time() - t0 > a.seconds:
            break
        c = draw(rng)
        try:
            out = run_case(o, c)
        except (spk.InvalidArgument, ValueError) as e:
            # plans the planner refuses (partition shorter than the band needs)
            rejected += 1
            c["rejected"] = str(e)[:100]
            print(json.dumps(c), flush=True)
            continue
        except Exception as e:  # anything else is a failure
            fails += 1
            c["error"] = f"{type(e).__name__}: {e}"[:300]
            print(json.dumps(c), flush=True)
            continue
        done += 1
        bad = False
        for key, (res, gap, ores) in out.items():
            if not (res <= RES_TOL and gap <= GAP_TOL) or not np.isfinite(gap):
                bad = True
            worst_res, worst_gap = max(worst_res, res), max(worst_gap, gap)
        if bad:
            fails += 1
            c["result"] = {k: [float(v) for v in vals] for k, vals in out.items()}
            print(json.dumps(c), flush=True)
    print(json.dumps({"summary": True, "cases_run": done, "failures": fails, "rejected_plans": rejected,
                      "worst_residual": worst_res, "worst_gap_dominant": worst_gap,
                      "seconds": round(time.time() - t0, 1), "seed": a.seed}), flush=True)
    sys.exit(1 if fails else 0)


if __name__ == "__main__":
    main()
