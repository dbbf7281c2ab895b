"""Verification and refinement on the device
against the C oracle (oracle/spike_oracle.c, itself pinned to the reference):

  band_matmul (tensor-core masked GEMM)   band_ops.cpp:11-37      -> oracle.matmul
  residual / backward error               band_ops.cpp:45-57      -> oracle.relative_residual, backward_error
  band norms                              band_ops.cpp:59-69      -> numpy on the packed band
  iterative_refine on the device          solve.cpp:404-432       -> the reference loop restated in numpy
  Hager condition estimate                oracle.cpp:132-166      -> oracle.cond1 (exact ||A||_1 ||A^-1||_1 bound)
"""
import numpy as np
import pytest
import torch

from conftest import rel_componentwise

pytestmark = pytest.mark.gpu


def dense(band, n, kl, ku):
    A = np.zeros((n, n))
    for j in range(n):
        for i in range(max(0, j - ku), min(n, j + kl + 1)):
            A[i, j] = band[j, ku + i - j]
    return A


@pytest.mark.parametrize("n,kl,ku,nc", [(1, 0, 0, 1), (70, 3, 5, 2), (500, 16, 16, 65), (1000, 7, 2, 1),
                                        (3000, 40, 40, 130), (129, 64, 1, 3)])
@pytest.mark.parametrize("tr", [False, True])
def test_band_matmul_matches_oracle(oracle, spk, n, kl, ku, nc, tr):
    band = oracle.generate_band(300 + n + kl, n, kl, ku, 1.3)
    X = np.asfortranarray(oracle.generate_rhs(301 + n, n, nc))
    a = spk.BandedMatrix(n, kl, ku, band)
    y = spk.band_matmul(a, X, tr)
    want = oracle.matmul(band, n, kl, ku, X, tr)
    assert rel_componentwise(y, want) <= 1e-14
    if n <= 500:
        A = dense(band, n, kl, ku)
        assert rel_componentwise(y, (A.T if tr else A) @ X) <= 1e-14


@pytest.mark.parametrize("tr", [False, True])
def test_residual_norms_and_backward_error(oracle, spk, tr):
    n, kl, ku, nc = 20000, 9, 12, 7
    band = oracle.generate_band(77, n, kl, ku, 1.4)
    F = np.asfortranarray(oracle.generate_rhs(78, n, nc))
    a = spk.BandedMatrix(n, kl, ku, band)
    fact = spk.factorize(a, spk.gpu_plan(n, kl, ku, nc, False, 9))
    X = spk.transpose_solve(fact, F) if tr else spk.solve(fact, F)
    dev = torch.device("cuda", 0)
    db = torch.from_numpy(np.ascontiguousarray(band)).to(dev)
    dX0 = torch.from_numpy(np.ascontiguousarray(X.T)).to(dev)
    dF0 = torch.from_numpy(np.ascontiguousarray(F.T)).to(dev)
    assert spk.backward_error_device(db.data_ptr(), n, kl, ku, dX0.data_ptr(), n, dF0.data_ptr(), n, nc, tr) <= 1e-12
    # a perturbed X: residuals well above rounding, so the statistics compare meaningfully
    X = np.asfortranarray(X + 1e-3 * oracle.generate_rhs(79, n, nc))
    dX = torch.from_numpy(np.ascontiguousarray(X.T)).to(dev)
    dF = torch.from_numpy(np.ascontiguousarray(F.T)).to(dev)
    dR = torch.empty_like(dF)
    st = spk.residual_device(db.data_ptr(), n, kl, ku, dX.data_ptr(), n, dF.data_ptr(), n, nc, tr, dR.data_ptr(), n)
    torch.cuda.synchronize()
    R = dR.cpu().numpy().T
    want_R = F - oracle.matmul(band, n, kl, ku, X, tr)
    assert np.abs(R - want_R).max() <= 1e-14 * np.abs(F).max()
    assert np.allclose(st[:, 0], (R ** 2).sum(axis=0), rtol=1e-12, atol=0)
    assert np.allclose(st[:, 1], (F ** 2).sum(axis=0), rtol=1e-12, atol=0)
    assert np.array_equal(st[:, 2], np.abs(R).max(axis=0))
    assert np.array_equal(st[:, 3], np.abs(X).max(axis=0))
    # Frobenius relative residual and the normwise backward error (SURVEY 8(d) i, iii)
    rr = np.sqrt(st[:, 0].sum()) / np.sqrt(st[:, 1].sum())
    assert abs(rr - oracle.relative_residual(band, n, kl, ku, X, F, tr)) <= 1e-12 * rr
    be = spk.backward_error_device(db.data_ptr(), n, kl, ku, dX.data_ptr(), n, dF.data_ptr(), n, nc, tr)
    bo = oracle.backward_error(band, n, kl, ku, X, F, tr)
    assert abs(be - bo) <= 1e-12 * bo


@pytest.mark.parametrize("n,kl,ku", [(1, 0, 0), (1000, 5, 9), (4097, 33, 2)])
def test_band_norms(oracle, spk, n, kl, ku):
    band = oracle.generate_band(55 + n, n, kl, ku, 1.2)
    db = torch.from_numpy(np.ascontiguousarray(band)).cuda()
    n1, ninf, mx = spk.band_norms_device(db.data_ptr(), n, kl, ku)
    A = np.abs(dense(band, n, kl, ku))
    assert abs(n1 - A.sum(axis=0).max()) <= 1e-14 * n1
    assert abs(ninf - A.sum(axis=1).max()) <= 1e-14 * ninf
    assert mx == A.max()


def refine_numpy(spk, fact, a, F, x0, max_iters, tol, tr):
    """solve.cpp:404-432 restated (host loop, GPU solves), the reference semantics."""
    x = x0.copy()
    fnorm = np.linalg.norm(F)
    prev = np.inf
    for it in range(max_iters + 1):
        r = F - spk.band_matmul(a, x, tr)
        rn = np.linalg.norm(r)
        res = (0.0 if rn == 0 else np.inf) if fnorm == 0 else rn / fnorm
        if res <= tol:
            return x, it, res, True, False
        if it > 0 and res * 1.1 > prev:
            return x, it, res, False, True
        if it == max_iters:
            return x, it, res, False, False
        prev = res
        x = x + (spk.transpose_solve(fact, r) if tr else spk.solve(fact, r))


@pytest.mark.parametrize("tr", [False, True])
@pytest.mark.parametrize("max_iters,tol", [(5, 1e-13), (0, 1e-13), (8, 0.0)])
def test_refine_device_matches_reference_loop(oracle, spk, tr, max_iters, tol):
    """A boosted (non-pivoting, zero pivot) factorization refined on the device."""
    n, k, nc = 3000, 4, 3
    band = oracle.generate_band(91, n, k, k, 1.5)
    F = np.asfortranarray(oracle.generate_rhs(92, n, nc))
    a = spk.BandedMatrix(n, k, k, band)
    a.set(0, 0, 0.0)
    a.set(1500, 1500, 0.0)
    fact = spk.factorize(a, spk.gpu_plan(n, k, k, nc, False, 6))
    assert fact.boost_count >= 1
    x0 = np.zeros((n, nc), order="F")
    got = spk.iterative_refine(fact, a, F, x0, max_iters, tol, tr)
    xw, itw, resw, convw, stagw = refine_numpy(spk, fact, a, F, x0, max_iters, tol, tr)
    assert (got.iterations, got.converged, got.stagnated) == (itw, convw, stagw)
    assert abs(got.residual - resw) <= 1e-6 * resw + 1e-300
    assert rel_componentwise(got.x, xw) <= 1e-12
    if max_iters == 5:
        assert got.converged and got.residual <= 1e-13
    # device buffers: same loop, X refined in place
    dev = torch.device("cuda", 0)
    db = torch.from_numpy(np.ascontiguousarray(a.data)).to(dev)
    dF = torch.from_numpy(np.ascontiguousarray(F.T)).to(dev)
    dX = torch.zeros_like(dF)
    r2 = spk.refine_device(fact, db.data_ptr(), dF.data_ptr(), n, nc, dX.data_ptr(), n, max_iters, tol, tr)
    assert (r2.iterations, r2.converged, r2.stagnated, r2.residual) == \
        (got.iterations, got.converged, got.stagnated, got.residual)
    assert np.array_equal(dX.cpu().numpy().T, got.x)


@pytest.mark.parametrize("n,k,dd,piv", [(400, 3, 1.2, False), (2000, 8, 1.05, False), (600, 4, 1.2, True)])
def test_condition_estimate_matches_oracle(oracle, spk, n, k, dd, piv):
    band = oracle.generate_band(123 + n, n, k, k, dd)
    a = spk.BandedMatrix(n, k, k, band)
    fact = spk.factorize(a, spk.gpu_plan(n, k, k, 1, piv, 4), spk.FactorOptions(pivoting=piv))
    est = spk.condition_estimate_1norm(fact, a)
    want = oracle.cond1(band, n, k, k)
    assert abs(est - want) <= 1e-6 * want
    if n <= 2000:
        A = dense(band, n, k, k)
        exact = np.linalg.norm(A, 1) * np.linalg.norm(np.linalg.inv(A), 1)
        assert est <= exact * (1 + 1e-9) and est >= 0.1 * exact
