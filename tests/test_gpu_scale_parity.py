"""Parity at the BASELINE scale and on the wide-band kernel templates.

* test_baseline_parity_vs_reference: the five BASELINE configurations at full
  size.  The compiled, unmodified reference (oracle/_ref, built from
  /root/reference/proj/src by oracle/Makefile; it travels to the GPU box) runs
  its own CPU path -- make_plan(n, k, k, t, compute_ratios(1, nrhs, k)),
  factorize, solve, transpose_solve -- on the host cores, on the same seeded
  inputs the GPU generates in HBM (include/spike_b200_gen.h, bit-identical on
  both sides).  North-star bar:
    (i)  normwise backward error max_c ||A x_c - f_c||_inf / (||A||_inf ||x_c||_inf)
         <= 1e-12 for the GPU solution (||A||_1 for the transpose);
    (ii) ||x_gpu - x_ref||_inf / ||x_ref||_inf <= 1e-10 * kappa, kappa the Varah
         bound (1 + dd) / (dd - 1) * max_i s_i / min_i s_i (s_i the off-diagonal
         row abs-sum; forward solves of the row-dominant configs) or Hager's
         1-norm estimate (transposes, and C4, where it is also compared with the
         reference's condition_estimate_1norm, oracle.cpp:132-166).
  The observed values are printed (and appended to $SPK_PARITY_LOG as JSON).
* test_wide_band_templates_vs_oracle: every k_band_lu_dmma / sweep template
  the large-k configurations run (k = 65 .. 160, narrow to wide right-hand
  sides, non-pivoting and pivoting) against the serial banded GE oracle.
* test_boosted_factorization_matches_reference: the golden boosted case
  (tests/golden/make_golden.py): same boost count as the reference, same
  boosted solution, and the device iterative_refine against the reference's
  iterative_refine on its own factorization.
"""
import json
import math
import os
import time

import numpy as np
import pytest

from conftest import rel_componentwise

pytestmark = pytest.mark.gpu

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "golden.npz")
BOOST_TOL = 1e-8  # see tests/test_oracle_golden.py


# name: n, k, nrhs, dd (<= 0: no dominance), pivoting, reference threads (None: all host cores)
BASELINE = {
    "C1": (100_000, 16, 1, 2.0, False, 4),
    "C2": (1_000_000, 64, 1, 1.1, False, 3),
    "C3": (1_000_000, 160, 160, 1.5, False, None),
    "C4": (1_000_000, 64, 4, -1.0, True, None),
    "C5": (16_000_000, 128, 32, 1.2, False, None),
}
SEED_A, SEED_F = 20181108, 20181109


def _row_offdiag_sums(band, n, k):
    """s_i = sum_{j != i} |a_ij| on the device; band is (n, 2k+1): packed row q
    of column j holds A(j + q - k, j)."""
    import torch
    absb = band.abs()
    s = torch.zeros(n, dtype=torch.float64, device=band.device)
    idx = torch.arange(n, device=band.device)
    for q in range(2 * k + 1):
        if q == k:
            continue
        i = idx + q - k
        ok = (i >= 0) & (i < n)
        s.index_add_(0, i[ok], absb[ok, q])
    return s


def _log(rec):
    path = os.environ.get("SPK_PARITY_LOG")
    print(json.dumps(rec))
    if path:
        with open(path, "a") as fp:
            fp.write(json.dumps(rec) + "\n")


@pytest.mark.slow
@pytest.mark.parametrize("cfg", sorted(BASELINE))
def test_baseline_parity_vs_reference(spk, reference, cfg):
    import torch
    if reference is None:
        pytest.skip("oracle/_ref (compiled reference) not built")
    n, k, nrhs, dd, piv, t = BASELINE[cfg]
    t = t or reference.L.ref_hw_threads()
    dev = torch.device("cuda", 0)
    s = torch.cuda.current_stream().cuda_stream
    band = torch.empty((n, 2 * k + 1), dtype=torch.float64, device=dev)
    F = torch.empty((nrhs, n), dtype=torch.float64, device=dev)  # column-major n x nrhs
    spk.generate_band_device(SEED_A, n, k, k, dd, band.data_ptr(), s)
    spk.generate_rhs_device(SEED_F, n, nrhs, F.data_ptr(), n, s)
    torch.cuda.synchronize()
    rec = {"cfg": cfg, "n": n, "k": k, "nrhs": nrhs, "pivoting": piv, "ref_threads": t}

    # GPU: the device plan, device-resident inputs
    plan = spk.gpu_plan(n, k, k, nrhs, piv)
    fact = spk.factorize_device(band.data_ptr(), n, k, k, plan, spk.FactorOptions(pivoting=piv), s)
    X = {tr: torch.empty_like(F) for tr in (False, True)}
    for tr in (False, True):
        spk.solve_device(fact, F.data_ptr(), n, nrhs, X[tr].data_ptr(), n, tr, s)
    torch.cuda.synchronize()
    rec["gpu_p"] = plan.p
    cond1 = spk.condition_estimate_device(fact, band.data_ptr(), s)
    rec["kappa1_hager_gpu"] = cond1
    del fact
    spk.lib().spk_arena_trim()  # C5: hand the factorization's HBM back before the checks

    # the reference CPU path on the same inputs
    hband = band.cpu().numpy()
    hF = F.cpu().numpy().T  # n x nrhs (F-ordered view)
    t0 = time.perf_counter()
    out = reference.time_path(hband, n, k, k, hF, t, 1.0, piv, True, want_x=True)
    rec["ref_wall_s"] = round(time.perf_counter() - t0, 2)
    rec["ref_p"] = out["p"]
    rec["ref_times_s"] = [out["factor"], out["solve"], out["tsolve"]]
    XR = {False: torch.from_numpy(np.ascontiguousarray(out["X"].T)).to(dev),
          True: torch.from_numpy(np.ascontiguousarray(out["XT"].T)).to(dev)}
    del out, hF

    if dd > 0:
        srow = _row_offdiag_sums(band, n, k)
        varah = (1.0 + dd) / (dd - 1.0) * (srow.max() / srow.min()).item()
        rec["kappa_inf_varah"] = varah
        del srow
    if piv:
        kref = reference.cond1(hband, n, k, k)
        rec["kappa1_hager_ref"] = kref
        assert 0.5 <= cond1 / kref <= 2.0, (cond1, kref)
    del hband

    for tr in (False, True):
        tag = "transpose" if tr else "forward"
        be = spk.backward_error_device(band.data_ptr(), n, k, k, X[tr].data_ptr(), n, F.data_ptr(), n, nrhs, tr, s)
        be_ref = spk.backward_error_device(band.data_ptr(), n, k, k, XR[tr].data_ptr(), n, F.data_ptr(), n, nrhs,
                                           tr, s)
        dx = ((X[tr] - XR[tr]).abs().max() / XR[tr].abs().max()).item()
        kappa = rec["kappa_inf_varah"] if (dd > 0 and not tr) else cond1
        rec[tag] = {"backward_error_gpu": be, "backward_error_ref": be_ref, "dx_rel_inf": dx,
                    "kappa": kappa, "dx_bound": 1e-10 * kappa}
        assert be <= 1e-12, (cfg, tag, be)
        assert dx <= 1e-10 * kappa, (cfg, tag, dx, kappa)
    _log(rec)


# k: every non-pivoting DMMA LU template (<13,13> k <= 96, <17,17> k <= 128,
# <21,12> k <= 160) and sweep window (NTW 9 .. 21); nrhs 1 (paired narrow
# sweeps), 33 (k_sweep_dmma warp pairs), 160 (k_sweep_dmma2 producer/consumer)
WIDE = [(k, nrhs, piv) for k in (65, 96, 128, 160) for nrhs in (1, 33, 160) for piv in (False, True)]


@pytest.mark.parametrize("k,nrhs,piv", WIDE)
def test_wide_band_templates_vs_oracle(oracle, spk, k, nrhs, piv):
    n = 30000
    band = oracle.generate_band(5000 + k + nrhs, n, k, k, 1.5)
    F = np.asfortranarray(oracle.generate_rhs(5001 + k, n, nrhs))
    a = spk.BandedMatrix(n, k, k, band)
    for plan in (spk.gpu_plan(n, k, k, nrhs, piv), spk.gpu_plan(n, k, k, nrhs, piv, 13)):
        fact = spk.factorize(a, plan, spk.FactorOptions(pivoting=piv))
        for tr in (False, True):
            X = spk.transpose_solve(fact, F) if tr else spk.solve(fact, F)
            Xo = oracle.oracle_solve(band, n, k, k, F, tr, True)
            res = oracle.relative_residual(band, n, k, k, X, F, tr)
            gap = rel_componentwise(X, Xo)
            assert res <= 1e-12 and gap <= 1e-10, (plan.p, tr, res, gap)
    # every stage on a tuned kernel, except the pivoted transposed L sweep of
    # bands with kl + ku > 192: no blocked L records there (the pivoted DMMA
    # LU's window needs one warp per 8 columns), so it runs the generic kernel
    gen = spk.generic_launch_count(reset=True)
    assert gen == 0 or (piv and 2 * k > 192), gen


def test_boosted_factorization_matches_reference(spk):
    g = np.load(GOLD)
    n, kl, ku, nrhs, t, piv = [int(x) for x in g["boost/shape"]]
    band = np.ascontiguousarray(g["boost/band"])
    F = np.asfortranarray(g["boost/F"])
    bounds = [int(b) for b in g["boost/bounds"]]
    kinds = [spk.PartitionKind.FirstLast] + [spk.PartitionKind.InnerSingle] * (len(bounds) - 3) + \
        [spk.PartitionKind.FirstLast]
    plan = spk.PartitionPlan(p=len(bounds) - 1, bounds=bounds, kinds=kinds)
    a = spk.BandedMatrix(n, kl, ku, band)
    fact = spk.factorize(a, plan)
    assert fact.boost_count == int(g["boost/boost_count"][0])
    assert rel_componentwise(spk.solve(fact, F), g["boost/x"]) <= BOOST_TOL
    assert rel_componentwise(spk.transpose_solve(fact, F), g["boost/xt"]) <= BOOST_TOL
    for tr, key in ((False, "x_refined"), (True, "xt_refined")):
        its, conv, stag, res = g["boost/refine"][int(tr)]
        r = spk.iterative_refine(fact, a, F, np.zeros((n, nrhs)), 10, 1e-14, tr)
        assert r.converged and bool(conv)
        assert abs(r.iterations - int(its)) <= 1, (r.iterations, its)
        assert rel_componentwise(r.x, g["boost/" + key]) <= 1e-12
        assert r.residual <= 1e-14
