"""Multi-GPU slab path (paper_1811_03559_b200/distributed.py) on one GPU.

Every slab is a real CUDA slab factorization (spk_factorize_slab /
spk_xsolve_*); the G ranks run as virtual ranks in one process, their
exchanges done by concatenation (``lockstep``) instead of NCCL, so no kernel
ever waits on another rank.  The assembled global X must solve the global
system like the single-GPU path and the oracle's banded GE (same tolerances as
test_gpu_parity.py).  The NCCL driver (``collective``) shares the per-rank
protocol; its host logic runs under gloo in test_distributed_host.py.
"""
import numpy as np
import pytest
import torch

from conftest import rel_componentwise

pytestmark = pytest.mark.gpu

RES_TOL = 1e-12
GAP_TOL = 1e-10


def run_virtual(spk, band_np, n, kl, ku, F_np, G, p_local, piv, dd_tol=True):
    from paper_1811_03559_b200 import distributed as D

    k = max(kl, ku)
    ld = kl + ku + 1
    dev = torch.device("cuda", 0)
    band = torch.from_numpy(np.ascontiguousarray(band_np)).to(dev)  # (n, ld): column j contiguous
    nrhs = F_np.shape[1]
    F = torch.from_numpy(np.ascontiguousarray(F_np.T)).to(dev)  # (nrhs, n) == column-major n x nrhs
    rows = D.slab_rows(n, G)
    opts = spk.FactorOptions(pivoting=piv)
    slabs = []
    for g in range(G):
        lh, _ = D.halo(g, G, k)
        ng = rows[g + 1] - rows[g]
        plan = spk.gpu_plan(ng, kl, ku, nrhs, piv, p_local)
        ptr = band.data_ptr() + (rows[g] - lh) * ld * 8
        slabs.append(D.CudaSlab(ptr, ng, kl, ku, plan, g, G, opts))
    res = D.lockstep([D.factorize_steps(s, opts.boost_eps) for s in slabs])
    tops = [r[1] for r in res]
    out = {}
    for tr in (False, True):
        X = torch.full_like(F, float("nan"))
        for g, s in enumerate(slabs):
            s.bind(F.data_ptr() + rows[g] * 8, n, nrhs, X.data_ptr() + rows[g] * 8, n)
        D.lockstep([D.solve_steps(s, tops[g], tr) for g, s in enumerate(slabs)])
        torch.cuda.synchronize()
        out[tr] = np.asfortranarray(X.cpu().numpy().T)
    return out, slabs, tops


CASES = [
    # G, n, kl, ku, nrhs, p_local, piv
    (2, 3000, 8, 8, 3, 4, False),
    (2, 3000, 8, 8, 3, 1, False),
    (3, 5000, 10, 10, 2, 3, False),
    (4, 4000, 5, 5, 2, 1, False),
    (4, 8000, 16, 16, 17, 5, False),
    (3, 6000, 7, 4, 2, 4, False),
    (2, 4000, 3, 9, 5, 2, False),
    (5, 10000, 12, 12, 9, 7, False),
    (8, 16000, 6, 6, 3, 3, False),
    (2, 3000, 6, 6, 2, 5, True),
    (3, 4500, 5, 8, 2, 2, True),
    (4, 8000, 40, 40, 40, 3, False),
]


@pytest.mark.parametrize("G,n,kl,ku,nrhs,p_local,piv", CASES)
def test_virtual_ranks_match_oracle(oracle, spk, G, n, kl, ku, nrhs, p_local, piv):
    seed = 7000 + G * 13 + n + kl * 3 + ku + nrhs
    band = oracle.generate_band(seed, n, kl, ku, 1.5)
    F = np.asfortranarray(oracle.generate_rhs(seed + 1, n, nrhs))
    out, _, _ = run_virtual(spk, band, n, kl, ku, F, G, p_local, piv)
    for tr in (False, True):
        xo = oracle.oracle_solve(band, n, kl, ku, F, tr, True)
        res = oracle.relative_residual(band, n, kl, ku, out[tr], F, tr)
        gap = rel_componentwise(out[tr], xo)
        assert res <= RES_TOL, (tr, res)
        assert gap <= GAP_TOL, (tr, gap)


def test_virtual_ranks_match_single_gpu(oracle, spk):
    """Same global system: G slabs vs one GPU factorization, agreement to
    rounding (different reduction trees, so not bit-identical)."""
    n, k, nrhs = 12000, 20, 24
    band = oracle.generate_band(4242, n, k, k, 1.2)
    F = np.asfortranarray(oracle.generate_rhs(4243, n, nrhs))
    a = spk.BandedMatrix(n, k, k, band)
    fact = spk.factorize(a, spk.gpu_plan(n, k, k, nrhs, False, 12))
    xs = {False: spk.solve(fact, F), True: spk.transpose_solve(fact, F)}
    out, _, _ = run_virtual(spk, band, n, k, k, F, 4, 3, False)
    for tr in (False, True):
        assert rel_componentwise(out[tr], xs[tr]) <= GAP_TOL


def test_slab_unit_tips_are_slab_spikes(oracle, spk):
    """The exchanged unit tips are the top/bottom k rows of the slab spikes
    V = A_g^-1 [0; bhat], W = A_g^-1 [chat; 0] (dense check on a small slab)."""
    from paper_1811_03559_b200 import distributed as D

    n, k, G = 600, 4, 3
    band = oracle.generate_band(99, n, k, k, 1.5)
    A = np.zeros((n, n))
    for j in range(n):
        for i in range(max(0, j - k), min(n, j + k + 1)):
            A[i, j] = band[j, k + i - j]
    F = np.asfortranarray(oracle.generate_rhs(100, n, 2))
    _, slabs, _ = run_virtual(spk, band, n, k, k, F, G, 3, False)
    rows = D.slab_rows(n, G)
    g = 1
    r0, r1 = rows[g], rows[g + 1]
    Ag = A[r0:r1, r0:r1]
    rhs_v = np.zeros((r1 - r0, k))
    rhs_v[-k:] = A[r1 - k:r1, r1:r1 + k]
    rhs_w = np.zeros((r1 - r0, k))
    rhs_w[:k] = A[r0:r0 + k, r0 - k:r0]
    V = np.linalg.solve(Ag, rhs_v)
    W = np.linalg.solve(Ag, rhs_w)
    tips = slabs[g].factor_tips().cpu().numpy().reshape(4, k, k).transpose(0, 2, 1)  # column-major blocks
    for got, want in zip(tips, (V[:k], V[-k:], W[:k], W[-k:])):
        assert np.abs(got - want).max() <= 1e-12 * max(1.0, np.abs(want).max())


def test_slab_rejects_closed_solve_api(oracle, spk):
    """A slab factorization needs the exchange protocol: spk_solve refuses it."""
    from paper_1811_03559_b200 import distributed as D

    n, k = 2000, 4
    band = oracle.generate_band(5, n, k, k, 1.5)
    F = np.asfortranarray(oracle.generate_rhs(6, n, 1))
    _, slabs, _ = run_virtual(spk, band, n, k, k, F, 2, 2, False)
    with pytest.raises(spk.InvalidArgument):
        spk.solve_device(slabs[0].fact, 0, slabs[0].n, 1, 0, slabs[0].n)
