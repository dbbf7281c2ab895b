"""The C++ multi-GPU data plane (csrc/spk_dist.cu) on one GPU.

* spk_dist_exchange -- the exchange arithmetic the library runs between its
  NCCL all-gathers -- against distributed.py's tensor formulas (the protocol
  the gloo tests run on the CPU), for several slab counts and ranks;
* the slab protocol over G virtual ranks with every exchange computed by the
  library kernels (no rank waits on another: the gathers are concatenations),
  against the oracle's banded GE;
* spk_dist_factorize / spk_dist_solve with a real one-rank NCCL communicator
  (NcclPlane.single): the data plane's own collectives, against the
  single-GPU solve.  (Two NCCL ranks on one GPU are not allowed; the
  multi-rank plane runs under bench.py --gpus N.)
"""
import numpy as np
import pytest
import torch

from conftest import rel_componentwise

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("G", [1, 2, 3, 5])
@pytest.mark.parametrize("k,nrhs", [(4, 3), (16, 1), (7, 8)])
def test_exchange_kernels_match_tensor_formulas(spk, G, k, nrhs):
    from paper_1811_03559_b200 import distributed as D

    dev = torch.device("cuda", 0)
    gen = torch.Generator(device="cpu").manual_seed(G * 100 + k * 10 + nrhs)
    g2 = torch.randn(G, 2 * k * nrhs, generator=gen, dtype=torch.float64).to(dev)
    g4 = torch.randn(G, 4 * k * nrhs, generator=gen, dtype=torch.float64).to(dev)
    z = torch.randn(nrhs, 2 * G * k, generator=gen, dtype=torch.float64).to(dev)
    got = D.exchange_device(D.XCH_FWD_TOP_RHS, g2, G, 0, k, nrhs)
    assert torch.equal(got, D.forward_top_rhs(g2, k, nrhs).reshape(-1))
    got = D.exchange_device(D.XCH_TR_TOP_RHS, g4, G, 0, k, nrhs)
    assert torch.allclose(got, D.transpose_top_rhs(g4, k, nrhs).reshape(-1), rtol=0, atol=0)
    for rank in range(G):
        got = D.exchange_device(D.XCH_FWD_IMPORT, z, G, rank, k, nrhs)
        assert torch.equal(got, D.forward_import(z, rank, G, k).reshape(-1)), rank
        got = D.exchange_device(D.XCH_TR_IMPORT1, g2, G, rank, k, nrhs)
        assert torch.equal(got, D.transpose_import1(g2, rank, G, k, nrhs).reshape(-1)), rank
        got = D.exchange_device(D.XCH_TR_IMPORT2, z, G, rank, k, nrhs)
        assert torch.equal(got, D.transpose_import2(z, rank, G, k).reshape(-1)), rank


def _device_solve_steps(slab, top, transpose):
    """distributed.solve_steps with the library's exchange kernels."""
    from paper_1811_03559_b200 import distributed as D

    k, g, G, nrhs = slab.k, slab.rank, slab.world, slab.nrhs
    state, exp = slab.begin(transpose)
    gathered = yield exp
    if not transpose:
        z = D.exchange_device(D.XCH_FWD_TOP_RHS, gathered.contiguous(), G, g, k, nrhs).reshape(nrhs, 2 * G * k)
        slab.top_solve(top, False, z)
        slab.step(state, D.exchange_device(D.XCH_FWD_IMPORT, z, G, g, k, nrhs))
    else:
        exp2 = slab.step(state, D.exchange_device(D.XCH_TR_IMPORT1, gathered.contiguous(), G, g, k, nrhs))
        gathered = yield exp2
        z = D.exchange_device(D.XCH_TR_TOP_RHS, gathered.contiguous(), G, g, k, nrhs).reshape(nrhs, 2 * G * k)
        slab.top_solve(top, True, z)
        slab.step(state, D.exchange_device(D.XCH_TR_IMPORT2, z, G, g, k, nrhs))
    slab.end(state)


@pytest.mark.parametrize("G,n,kl,ku,nrhs,p_local,piv", [
    (2, 3000, 8, 8, 3, 4, False),
    (3, 6000, 12, 9, 5, 3, False),
    (4, 8000, 16, 16, 2, 2, False),
    (3, 4000, 6, 6, 2, 2, True),
])
def test_virtual_ranks_with_library_exchanges(oracle, spk, G, n, kl, ku, nrhs, p_local, piv):
    from paper_1811_03559_b200 import distributed as D

    k = max(kl, ku)
    ld = kl + ku + 1
    band_np = oracle.generate_band(700 + G + n, n, kl, ku, 1.5)
    F_np = np.asfortranarray(oracle.generate_rhs(701 + n, n, nrhs))
    dev = torch.device("cuda", 0)
    band = torch.from_numpy(np.ascontiguousarray(band_np)).to(dev)
    F = torch.from_numpy(np.ascontiguousarray(F_np.T)).to(dev)
    rows = D.slab_rows(n, G)
    opts = spk.FactorOptions(pivoting=piv)
    slabs = []
    for g in range(G):
        lh, _ = D.halo(g, G, k)
        ng = rows[g + 1] - rows[g]
        plan = spk.gpu_plan(ng, kl, ku, nrhs, piv, p_local)
        slabs.append(D.CudaSlab(band.data_ptr() + (rows[g] - lh) * ld * 8, ng, kl, ku, plan, g, G, opts))
    res = D.lockstep([D.factorize_steps(s, opts.boost_eps) for s in slabs])
    tops = [r[1] for r in res]
    for tr in (False, True):
        X = torch.full_like(F, float("nan"))
        for g, s in enumerate(slabs):
            s.bind(F.data_ptr() + rows[g] * 8, n, nrhs, X.data_ptr() + rows[g] * 8, n)
        D.lockstep([_device_solve_steps(s, tops[g], tr) for g, s in enumerate(slabs)])
        torch.cuda.synchronize()
        Xh = np.asfortranarray(X.cpu().numpy().T)
        Xo = oracle.oracle_solve(band_np, n, kl, ku, F_np, tr, True)
        res_ = oracle.relative_residual(band_np, n, kl, ku, Xh, F_np, tr)
        assert res_ <= 1e-12, (tr, res_)
        assert rel_componentwise(Xh, Xo) <= (1e-8 if piv else 1e-10), tr


@pytest.mark.parametrize("kl,ku,nrhs,piv", [(16, 16, 3, False), (40, 33, 8, False), (24, 24, 2, True)])
def test_nccl_plane_single_rank(oracle, spk, kl, ku, nrhs, piv):
    from paper_1811_03559_b200 import distributed as D

    n = 20000
    band_np = oracle.generate_band(808 + kl, n, kl, ku, -1.0 if piv else 1.5)
    F_np = np.asfortranarray(oracle.generate_rhs(809, n, nrhs))
    dev = torch.device("cuda", 0)
    band = torch.from_numpy(np.ascontiguousarray(band_np)).to(dev)
    F = torch.from_numpy(np.ascontiguousarray(F_np.T)).to(dev)
    plane = D.NcclPlane.single()
    plan = spk.gpu_plan(n, kl, ku, nrhs, piv, 0)
    s = torch.cuda.current_stream().cuda_stream
    df = plane.factorize(band.data_ptr(), n, kl, ku, plan, spk.FactorOptions(pivoting=piv), s)
    ref = spk.factorize(spk.BandedMatrix(n, kl, ku, band_np), plan, spk.FactorOptions(pivoting=piv))
    for tr in (False, True):
        X = torch.full_like(F, float("nan"))
        plane.solve(df, F.data_ptr(), n, nrhs, X.data_ptr(), n, tr, s)
        torch.cuda.synchronize()
        Xh = np.asfortranarray(X.cpu().numpy().T)
        Xr = spk.transpose_solve(ref, F_np) if tr else spk.solve(ref, F_np)
        assert np.array_equal(Xh, Xr), tr
