"""Stream-ordered C-ABI and the generic coupling path.

* spk_factorize returns once enqueued; a host-memory spk_solve issued right
  after it runs the device-guarded solve programs (coupling paths decided on
  the device) and returns before X lands; spk_stream_sync completes it.  The
  result must equal the synchronous path's (unguarded programs) bit for bit.
* Reduced systems whose W blocks exceed 1 in magnitude take the generic 2k
  coupling path (pivoted coupling LU, reference factorize.cpp:94-102) instead
  of the Schur complement; checked against a dense solve.
"""
import ctypes as C

import numpy as np
import pytest
import torch

from conftest import rel_componentwise

pytestmark = pytest.mark.gpu


def _reduced_dense(vt, vb, wt, wb, p, k):
    N = 2 * p * k
    red = np.eye(N)
    for i in range(p):
        if i + 1 < p:
            red[2 * i * k:(2 * i + 1) * k, 2 * (i + 1) * k:(2 * i + 3) * k] = vt[i]
            red[(2 * i + 1) * k:(2 * i + 2) * k, 2 * (i + 1) * k:(2 * i + 3) * k] = vb[i]
        if i > 0:
            red[2 * i * k:(2 * i + 1) * k, (2 * i - 1) * k:2 * i * k] = wt[i]
            red[(2 * i + 1) * k:(2 * i + 2) * k, (2 * i - 1) * k:2 * i * k] = wb[i]
    return red


@pytest.mark.parametrize("p", [2, 3, 5, 8])
@pytest.mark.parametrize("k", [1, 3, 8])
@pytest.mark.parametrize("scale", [0.4, 3.0])
def test_reduced_generic_and_schur_paths(spk, p, k, scale):
    """scale 3: |W| > 1 in most pairs (generic path); 0.4: Schur path."""
    rng = np.random.default_rng(900 + 31 * p + k + int(10 * scale))
    vt, vb, wt, wb = [[scale * (rng.random((k, k)) - 0.5) for _ in range(p)] for _ in range(4)]
    red = _reduced_dense(vt, vb, wt, wb, p, k)
    if np.linalg.cond(red) > 1e8:
        pytest.skip("ill-conditioned draw")
    rl = spk.reduce_factorize(vt, vb, wt, wb, p, k)
    y = rng.random((2 * p * k, 3))
    x = spk.reduced_solve(rl, y, [])
    xt = spk.reduced_solve_transpose(rl, y, [])
    tol = 1e-13 * max(1.0, np.linalg.cond(red))
    assert rel_componentwise(x, np.linalg.solve(red, y)) <= tol
    assert rel_componentwise(xt, np.linalg.solve(red.T, y)) <= tol


CASES = [
    # n, k, nrhs, p, dd, piv
    (20000, 8, 40, 9, 1.3, False),
    (20000, 5, 33, 6, 1.2, True),
    (12000, 6, 48, 7, 0.6, True),  # not dominant: generic coupling pairs
    (30000, 40, 64, 5, 1.5, False),
]


@pytest.mark.parametrize("n,k,nrhs,p,dd,piv", CASES)
def test_stream_ordered_host_solve_matches_sync(oracle, spk, n, k, nrhs, p, dd, piv):
    L = spk.lib()
    band = oracle.generate_band(4000 + n + k, n, k, k, dd)
    F = np.asfortranarray(oracle.generate_rhs(4001 + n, n, nrhs))
    plan = spk.gpu_plan(n, k, k, nrhs, piv, p)
    opts = spk.FactorOptions(pivoting=piv)
    # synchronous reference: the Python API (factorize waits, unguarded programs)
    a = spk.BandedMatrix(n, k, k, band)
    fact = spk.factorize(a, plan, opts)
    want = {False: spk.solve(fact, F), True: spk.transpose_solve(fact, F)}
    # stream-ordered raw C-ABI with pinned host buffers
    hband = torch.from_numpy(np.ascontiguousarray(band)).pin_memory()
    hF = torch.from_numpy(np.ascontiguousarray(F.T)).pin_memory()  # column-major n x nrhs
    hX = {tr: torch.full_like(hF, float("nan")).pin_memory() for tr in (False, True)}
    st, keep = spk.spike._plan_struct(plan)
    o = spk.spike._Opts(int(piv), opts.boost_eps)
    h = C.c_void_p()
    spk.spike._check(L.spk_factorize(C.c_void_p(hband.data_ptr()), 0, n, k, k, C.byref(st), C.byref(o), None,
                                     C.byref(h)))
    try:
        for tr in (False, True):
            spk.spike._check(L.spk_solve(h, int(tr), C.c_void_p(hF.data_ptr()), n, nrhs,
                                         C.c_void_p(hX[tr].data_ptr()), n, 0, None, None))
        spk.spike._check(L.spk_stream_sync(None))
        spk.spike._check(L.spk_fact_sync(h))
    finally:
        L.spk_fact_destroy(h)
    for tr in (False, True):
        got = hX[tr].numpy().T
        assert np.array_equal(got, want[tr]), (tr, rel_componentwise(got, want[tr]))


def test_singular_reported_by_fact_sync(spk):
    """Pivoting mode, exactly zero column: the stream-ordered factorization
    reports SPK_ESINGULAR at spk_fact_sync (the reference throws at factorize);
    the raw C-ABI call itself returns once enqueued."""
    n, k = 4000, 3
    a = spk.BandedMatrix(n, k, k)
    for i in range(n):
        a.set(i, i, 2.0)
    for i in range(1234 - k, 1234 + k + 1):
        a.set(i, 1234, 0.0)
    plan = spk.gpu_plan(n, k, k, 1, True, 4)
    with pytest.raises(RuntimeError):
        spk.factorize(a, plan, spk.FactorOptions(pivoting=True))
    L = spk.lib()
    st, keep = spk.spike._plan_struct(plan)
    o = spk.spike._Opts(1, spk.FactorOptions().boost_eps)
    h = C.c_void_p()
    band = np.ascontiguousarray(a.data)
    spk.spike._check(L.spk_factorize(C.c_void_p(band.ctypes.data), 0, n, k, k, C.byref(st), C.byref(o), None,
                                     C.byref(h)))
    try:
        assert L.spk_fact_sync(h) != 0
    finally:
        L.spk_fact_destroy(h)


def _raw_factorize(spk, band_ptr, mem, n, k, plan, piv, stream):
    L = spk.lib()
    st, keep = spk.spike._plan_struct(plan)
    o = spk.spike._Opts(int(piv), spk.FactorOptions().boost_eps)
    h = C.c_void_p()
    spk.spike._check(L.spk_factorize(C.c_void_p(band_ptr), mem, n, k, k, C.byref(st), C.byref(o),
                                     C.c_void_p(stream), C.byref(h)))
    return h


@pytest.mark.parametrize("transpose", [False, True])
def test_solve_on_other_stream_orders_after_factorization(oracle, spk, transpose):
    """Factorize on stream A and solve device-resident on stream B right away
    (no host sync in between): the solve must wait for A's factor program and
    the upload of its solve jobs.  Destroying the factorization right after
    (a still-pending solve on B) must not let A's next allocations reuse the
    memory B is reading."""
    L = spk.lib()
    n, k, nrhs, p = 400000, 64, 8, 148
    band = oracle.generate_band(777, n, k, k, 1.2)
    F = np.asfortranarray(oracle.generate_rhs(778, n, nrhs))
    plan = spk.gpu_plan(n, k, k, nrhs, False, p)
    want = (spk.transpose_solve if transpose else spk.solve)(
        spk.factorize(spk.BandedMatrix(n, k, k, band), plan), F)
    sa, sb = torch.cuda.Stream(), torch.cuda.Stream()
    dband = torch.from_numpy(np.ascontiguousarray(band)).cuda()
    dF = torch.from_numpy(np.ascontiguousarray(F.T)).cuda()  # column-major n x nrhs
    dX = torch.full_like(dF, float("nan"))
    torch.cuda.synchronize()
    for rep in range(3):
        dX.fill_(float("nan"))
        torch.cuda.synchronize()
        h = _raw_factorize(spk, dband.data_ptr(), 1, n, k, plan, False, sa.cuda_stream)
        spk.spike._check(L.spk_solve(h, int(transpose), C.c_void_p(dF.data_ptr()), n, nrhs,
                                     C.c_void_p(dX.data_ptr()), n, 1, C.c_void_p(sb.cuda_stream), None))
        L.spk_fact_destroy(h)
        # A reuses the released blocks at once: a second factorization of another matrix
        other = torch.from_numpy(np.ascontiguousarray(oracle.generate_band(779, n, k, k, 1.2))).cuda()
        h2 = _raw_factorize(spk, other.data_ptr(), 1, n, k, plan, False, sa.cuda_stream)
        sb.synchronize()
        sa.synchronize()
        L.spk_fact_destroy(h2)
        got = dX.cpu().numpy().T
        assert rel_componentwise(got, want) <= 1e-13, rep


def test_concurrent_first_solves_on_pending_factorization(oracle, spk):
    """Two threads make the first solves on a freshly enqueued (pending) raw
    C-ABI handle: the host-side finish runs once, both get the synchronous
    path's result bit for bit."""
    import threading
    L = spk.lib()
    n, k, nrhs = 60000, 16, 4
    band = oracle.generate_band(811, n, k, k, 1.5)
    F = np.asfortranarray(oracle.generate_rhs(812, n, nrhs))
    plan = spk.gpu_plan(n, k, k, nrhs, False, 64)
    fact = spk.factorize(spk.BandedMatrix(n, k, k, band), plan)
    want = {False: spk.solve(fact, F), True: spk.transpose_solve(fact, F)}
    for rep in range(4):
        h = _raw_factorize(spk, np.ascontiguousarray(band).ctypes.data, 0, n, k, plan, False, 0)
        out, errs = {}, []

        def work(tr):
            try:
                x = np.zeros((n, nrhs), order="F")
                s = torch.cuda.Stream()
                spk.spike._check(L.spk_solve(h, int(tr), C.c_void_p(F.ctypes.data), n, nrhs,
                                             C.c_void_p(x.ctypes.data), n, 0, C.c_void_p(s.cuda_stream), None))
                s.synchronize()
                out[tr] = x
            except Exception as e:  # pragma: no cover - reported below
                errs.append(e)

        ts = [threading.Thread(target=work, args=(tr,)) for tr in (False, True)]
        for t in ts:
            t.start()
        for t in ts:
            t.join()
        L.spk_fact_destroy(h)
        assert not errs, errs
        for tr in (False, True):
            assert np.array_equal(out[tr], want[tr]), (rep, tr)


def test_singular_status_is_sticky(spk):
    """After the deferred finish reports SPK_ESINGULAR, every later consumer
    of the handle (solves, getters) reports it too."""
    n, k = 4000, 3
    a = spk.BandedMatrix(n, k, k)
    for i in range(n):
        a.set(i, i, 2.0)
    for i in range(1234 - k, 1234 + k + 1):
        a.set(i, 1234, 0.0)
    plan = spk.gpu_plan(n, k, k, 1, True, 4)
    L = spk.lib()
    band = np.ascontiguousarray(a.data)
    h = _raw_factorize(spk, band.ctypes.data, 0, n, k, plan, True, 0)
    try:
        F = np.ones((n, 1), order="F")
        X = np.zeros((n, 1), order="F")
        assert L.spk_fact_sync(h) == 2
        assert L.spk_fact_sync(h) == 2
        assert L.spk_solve(h, 0, C.c_void_p(F.ctypes.data), n, 1, C.c_void_p(X.ctypes.data), n, 0, None,
                           None) == 2
        assert b"singular" in L.spk_last_error()
    finally:
        L.spk_fact_destroy(h)


def test_null_handles_are_rejected(spk):
    L = spk.lib()
    assert L.spk_solve(None, 0, None, 10, 1, None, 10, 0, None, None) == 1
    assert L.spk_factorize(None, 0, 10, 1, 1, None, None, None, None) == 1
    assert L.spk_fact_sync(None) == 1


@pytest.mark.parametrize("piv", [False, True])
def test_generic_path_matches_tuned_kernels(oracle, spk, piv):
    """The generic kernels (spk_set_generic_path) are the correctness baseline
    of the tuned ones: same answers to rounding on one input; the tuned run
    launches no generic kernel on this shape."""
    n, k, nrhs = 30000, 24, 6
    band = oracle.generate_band(901, n, k, k, 1.4)
    F = oracle.generate_rhs(902, n, nrhs)
    plan = spk.gpu_plan(n, k, k, nrhs, piv, 20)
    a = spk.BandedMatrix(n, k, k, band)
    spk.generic_launch_count(reset=True)
    fact = spk.factorize(a, plan, spk.FactorOptions(pivoting=piv))
    tuned = [spk.solve(fact, F), spk.transpose_solve(fact, F)]
    assert spk.generic_launch_count(reset=True) == 0
    with spk.generic_path():
        gfact = spk.factorize(a, plan, spk.FactorOptions(pivoting=piv))
        gen = [spk.solve(gfact, F), spk.transpose_solve(gfact, F)]
    assert spk.generic_launch_count(reset=True) > 0
    for t, g in zip(tuned, gen):
        assert rel_componentwise(t, g) <= 1e-11


def test_row_major_copy_lazy_and_in_kernel_agree(oracle, spk):
    """The DMMA LU writes the row-major factor copy only for shapes that have
    met a transposed solve; the first factorization of a shape makes it on
    demand (k_transpose_factors).  Transposed solves through either copy are
    bit-identical and match the oracle; forward solves never need it."""
    n, kl, ku = 6000, 33, 29  # a shape no other test uses
    band = oracle.generate_band(515, n, kl, ku, 1.5)
    F = np.asfortranarray(oracle.generate_rhs(516, n, 5))
    a = spk.BandedMatrix(n, kl, ku, band)
    plan = spk.gpu_plan(n, kl, ku, 5, False, 7)
    f1 = spk.factorize(a, plan)  # first of its shape: the copy is made on demand
    y1 = spk.solve(f1, F)
    x1 = spk.transpose_solve(f1, F)
    f2 = spk.factorize(a, plan)  # the shape has met a transposed solve: the copy comes from the LU
    x2 = spk.transpose_solve(f2, F)
    xo = oracle.oracle_solve(band, n, kl, ku, F, True, True)
    assert rel_componentwise(x1, xo) <= 1e-10 and rel_componentwise(x2, xo) <= 1e-10
    assert np.array_equal(x1, x2)
    assert np.array_equal(y1, spk.solve(f2, F))
