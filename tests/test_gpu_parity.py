"""GPU parity tests: the sm_100a path against the CPU oracle (oracle/spike_oracle.c,
pinned to the reference by tests/golden/).  Modelled on the reference suites
(paths under /root/reference/proj/tests):

  test_acceptance.cpp:40-85   oracle-equivalence grid      -> test_oracle_grid
  test_acceptance.cpp:87-107  sweep-count parity           -> test_sweep_budgets
  test_acceptance.cpp:109-151 reduced brute force          -> test_reduced_brute_force
  test_factor_ds.cpp:142-182  tips vs per-partition oracle -> test_tips_match_oracle
  test_factor_ds.cpp:287-303  determinism                  -> test_deterministic
  test_solve_stage.cpp:*      identity, reuse, re-entrancy, empty RHS, asymmetric bands

Tolerances are the reference's: relative residual <= 1e-12 and componentwise
gap <= 1e-10 against the oracle solution (fp64 throughout).
"""
import threading

import numpy as np
import pytest

from conftest import rel_componentwise

pytestmark = pytest.mark.gpu

RES_TOL = 1e-12
GAP_TOL = 1e-10


def make_case(oracle, spk, n, kl, ku, dd, nrhs, seed):
    band = oracle.generate_band(seed, n, kl, ku, dd)
    F = oracle.generate_rhs(seed + 1, n, nrhs)
    return spk.BandedMatrix(n, kl, ku, band), band, np.asfortranarray(F)


def check_solution(oracle, band, n, kl, ku, X, F, tr, xo):
    res = oracle.relative_residual(band, n, kl, ku, X, F, tr)
    gap = rel_componentwise(X, xo)
    return res, gap


GRID = [(n, k, nrhs) for n in (64, 512, 4096) for k in (1, 4, 16) for nrhs in sorted({1, k, 3 * k})]


@pytest.mark.parametrize("n,k,nrhs", GRID)
def test_oracle_grid(oracle, spk, n, k, nrhs):
    a, band, F = make_case(oracle, spk, n, k, k, 1.5, nrhs, 1000 + n + 7 * k + nrhs)
    xf = oracle.oracle_solve(band, n, k, k, F, False, True)
    xt = oracle.oracle_solve(band, n, k, k, F, True, True)
    plans = []
    for t in (2, 3, 4, 6, 8, 12, 14):
        r12, r13 = spk.compute_ratios(1.0, nrhs, k)
        plans.append(spk.make_plan(n, k, k, t, r12, r13))
    for p in (3, 5, 7, 13):  # non-power-of-two GPU plans
        if n // p >= 2 * k + 1:
            plans.append(spk.gpu_plan(n, k, k, nrhs, False, p))
    worst = 0.0
    for plan in plans:
        for piv in (False, True):
            fact = spk.factorize(a, plan, spk.FactorOptions(pivoting=piv))
            for tr in (False, True):
                X = spk.transpose_solve(fact, F) if tr else spk.solve(fact, F)
                res, gap = check_solution(oracle, band, n, k, k, X, F, tr, xt if tr else xf)
                worst = max(worst, gap)
                assert res <= RES_TOL and gap <= GAP_TOL, (plan.p, piv, tr, res, gap)


@pytest.mark.parametrize("p", [2, 3, 4, 5, 8, 11])
@pytest.mark.parametrize("piv", [False, True])
def test_matches_oracle_spike_same_plan(oracle, spk, p, piv):
    """Same plan on GPU and in the CPU restatement: solutions agree to rounding."""
    n, k, nrhs = 3000, 6, 5
    a, band, F = make_case(oracle, spk, n, k, k, 1.3, nrhs, 77 + p)
    plan = spk.gpu_plan(n, k, k, nrhs, piv, p)
    of = oracle.factorize(band, n, k, k, plan.bounds, piv)
    fact = spk.factorize(a, plan, spk.FactorOptions(pivoting=piv))
    for tr in (False, True):
        xo, swo, cco = of.solve(F, tr)
        st = spk.SolveStats()
        X = spk.transpose_solve(fact, F, st) if tr else spk.solve(fact, F, st)
        assert rel_componentwise(X, xo) <= 1e-12
        assert st.partition_full_sweeps == swo
        assert st.reduced_coupling_solves == cco
    assert fact.factor_sweeps == of.factor_sweeps()
    assert fact.levels.levels() == of.levels


def test_tips_match_oracle(oracle, spk):
    n, k = 96, 2
    for piv in (False, True):
        for p in (4, 3):
            a, band, _ = make_case(oracle, spk, n, k, k, 1.5, 1, 11)
            plan = spk.gpu_plan(n, k, k, 1, piv, p)
            fact = spk.factorize(a, plan, spk.FactorOptions(pivoting=piv))
            of = oracle.factorize(band, n, k, k, plan.bounds, piv)
            for i in range(p):
                for name in ("vt", "vb", "wt", "wb", "bhat", "chat"):
                    g = getattr(fact, name)[i]
                    o = of.tip(name, i)
                    assert np.allclose(g, o, rtol=1e-12, atol=1e-14), (piv, p, i, name)


def test_tips_vs_partition_oracle_spikes(oracle, spk):
    """test_factor_ds.cpp:142-182 : tips equal A_i^-1 [0; bhat] / A_i^-1 [chat; 0]."""
    n, k = 120, 3
    a, band, _ = make_case(oracle, spk, n, k, k, 1.5, 1, 31)
    plan = spk.gpu_plan(n, k, k, 1, False, 5)
    fact = spk.factorize(a, plan)
    ld = 2 * k + 1
    for i in range(plan.p):
        r0, m = plan.bounds[i], plan.size(i)
        sub = band[r0:r0 + m].copy()
        for j in range(m):
            for q in range(ld):
                ii = j + q - k
                if ii < 0 or ii >= m:
                    sub[j, q] = 0.0
        if i + 1 < plan.p:
            rhs = np.zeros((m, k), order="F")
            rhs[m - k:] = fact.bhat[i]
            v = oracle.oracle_solve(sub, m, k, k, rhs)
            if i > 0:
                assert np.allclose(fact.vt[i], v[:k], rtol=1e-12, atol=1e-15)
            assert np.allclose(fact.vb[i], v[m - k:], rtol=1e-12, atol=1e-15)
        if i > 0:
            rhs = np.zeros((m, k), order="F")
            rhs[:k] = fact.chat[i]
            w = oracle.oracle_solve(sub, m, k, k, rhs)
            assert np.allclose(fact.wt[i], w[:k], rtol=1e-12, atol=1e-15)
            if i + 1 < plan.p:
                assert np.allclose(fact.wb[i], w[m - k:], rtol=1e-12, atol=1e-15)


def test_sweep_budgets(oracle, spk):
    """test_acceptance.cpp:87-107 / test_solve_stage.cpp:196-216."""
    n, k = 2048, 8
    a, band, F = make_case(oracle, spk, n, k, k, 1.5, 3, 77)
    for t in (4, 5, 6, 8, 10, 12, 14):
        plan = spk.make_plan(n, k, k, t, 1.0, 2.0)
        for piv in (False, True):
            fact = spk.factorize(a, plan, spk.FactorOptions(pivoting=piv))
            st = spk.SolveStats()
            spk.solve(fact, F, st)
            for i in range(plan.p):
                boundary = plan.kinds[i] == spk.PartitionKind.FirstLast
                assert fact.factor_sweeps[i] == (0 if boundary else 3)
                assert st.partition_full_sweeps[i] == (2 if boundary else 4)
            assert st.reduced_coupling_solves == plan.p - 1


@pytest.mark.parametrize("p", [2, 3, 4, 5, 7, 8])
@pytest.mark.parametrize("k", [1, 2, 3])
def test_reduced_brute_force(oracle, spk, p, k):
    """test_acceptance.cpp:109-151 extended to non-power-of-two p."""
    rng = np.random.default_rng(4242 + 10 * p + k)
    vt, vb, wt, wb = [[rng.random((k, k)) - 0.5 for _ in range(p)] for _ in range(4)]
    rl = spk.reduce_factorize(vt, vb, wt, wb, p, k)
    N = 2 * p * k
    red = np.eye(N)
    for i in range(p):
        for c in range(k):
            for r in range(k):
                if i + 1 < p:
                    red[2 * i * k + r, 2 * (i + 1) * k + c] = vt[i][r, c]
                    red[(2 * i + 1) * k + r, 2 * (i + 1) * k + c] = vb[i][r, c]
                if i > 0:
                    red[2 * i * k + r, (2 * i - 1) * k + c] = wt[i][r, c]
                    red[(2 * i + 1) * k + r, (2 * i - 1) * k + c] = wb[i][r, c]
    y = rng.random((N, 2))
    cf, ct = [], []
    x = spk.reduced_solve(rl, y, cf)
    xt = spk.reduced_solve_transpose(rl, y, ct)
    assert cf == [p - 1] and ct == [p - 1]
    assert rel_componentwise(x, np.linalg.solve(red, y)) <= 1e-13
    assert rel_componentwise(xt, np.linalg.solve(red.T, y)) <= 1e-13
    # the C restatement agrees as well
    pack = lambda bl: np.ascontiguousarray(np.stack([b.T for b in bl]))
    zo, _ = oracle.reduced_solve_tips(pack(vt), pack(vb), pack(wt), pack(wb), p, k, y)
    assert rel_componentwise(x, zo) <= 1e-13


def test_identity_returns_f(spk):
    a = spk.BandedMatrix(32, 1, 1)
    for i in range(32):
        a.set(i, i, 1.0)
    plan = spk.make_plan(32, 1, 1, 4, 1.0, 2.0)
    fact = spk.factorize(a, plan)
    F = np.random.default_rng(3).random((32, 2))
    assert np.abs(spk.solve(fact, F) - F).max() == 0.0
    assert np.abs(spk.transpose_solve(fact, F) - F).max() == 0.0


def test_identity_factorization_trivial(spk):
    a = spk.BandedMatrix(64, 2, 2)
    for i in range(64):
        a.set(i, i, 1.0)
    for t in (2, 4, 6):
        fact = spk.factorize(a, spk.make_plan(64, 2, 2, t, 1.0, 2.0))
        for i in range(fact.p()):
            for name in ("vt", "vb", "wt", "wb"):
                assert np.abs(getattr(fact, name)[i]).max() == 0.0
        for level in fact.levels.pairs:
            for blk in level:
                for i in range(2 * fact.k):
                    assert blk.uval(i, i) == 1.0


def test_deterministic(oracle, spk):
    n, k = 256, 3
    a, band, F = make_case(oracle, spk, n, k, k, 1.5, 3, 31)
    plan = spk.make_plan(n, k, k, 6, 1.15, 2.3)
    f1 = spk.factorize(a, plan)
    f2 = spk.factorize(a, plan)
    for name in ("vt", "vb", "wt", "wb"):
        for x, y in zip(getattr(f1, name), getattr(f2, name)):
            assert np.array_equal(x, y)
    for l in range(f1.levels.levels()):
        for x, y in zip(f1.levels.v[l], f2.levels.v[l]):
            assert np.array_equal(x, y)
    assert np.array_equal(spk.solve(f1, F), spk.solve(f2, F))
    assert np.array_equal(spk.solve(f1, F), spk.solve(f1, F))


def test_transpose_reuse_and_symmetric(oracle, spk):
    n, k = 120, 2
    rng = np.random.default_rng(41)
    a = spk.BandedMatrix(n, k, k)
    for j in range(n):
        for i in range(j + 1, min(n, j + k + 1)):
            v = rng.random()
            a.set(i, j, v)
            a.set(j, i, v)
        a.set(j, j, 5.0)
    fact = spk.factorize(a, spk.make_plan(n, k, k, 4, 1.0, 2.0))
    F = rng.random((n, 2))
    assert np.abs(spk.solve(fact, F) - spk.transpose_solve(fact, F)).max() < 1e-13


def test_asymmetric_bands(oracle, spk):
    n, kl, ku = 300, 2, 5
    a, band, F = make_case(oracle, spk, n, kl, ku, 1.5, 3, 121)
    xf = oracle.oracle_solve(band, n, kl, ku, F, False, True)
    xt = oracle.oracle_solve(band, n, kl, ku, F, True, True)
    for t in (2, 4, 6):
        plan = spk.make_plan(n, kl, ku, t, 1.0, 2.0)
        for piv in (False, True):
            fact = spk.factorize(a, plan, spk.FactorOptions(pivoting=piv))
            assert rel_componentwise(spk.solve(fact, F), xf) < 1e-10
            assert rel_componentwise(spk.transpose_solve(fact, F), xt) < 1e-10
    plan = spk.gpu_plan(n, kl, ku, 3, False, 5)
    fact = spk.factorize(a, plan)
    assert rel_componentwise(spk.solve(fact, F), xf) < 1e-10
    assert rel_componentwise(spk.transpose_solve(fact, F), xt) < 1e-10


def test_concurrent_solves_reentrant(oracle, spk):
    n, k = 512, 4
    a, band, _ = make_case(oracle, spk, n, k, k, 1.5, 1, 111)
    fact = spk.factorize(a, spk.make_plan(n, k, k, 4, 1.0, 2.0))
    rng = np.random.default_rng(112)
    f1, f2 = rng.random((n, 2)), rng.random((n, 2))
    ref1, ref2 = spk.solve(fact, f1), spk.transpose_solve(fact, f2)
    out = {}
    t1 = threading.Thread(target=lambda: out.__setitem__(1, spk.solve(fact, f1)))
    t2 = threading.Thread(target=lambda: out.__setitem__(2, spk.transpose_solve(fact, f2)))
    t1.start(), t2.start(), t1.join(), t2.join()
    assert np.array_equal(out[1], ref1) and np.array_equal(out[2], ref2)


def test_empty_rhs_and_shape_errors(oracle, spk):
    n, k = 64, 2
    a, band, _ = make_case(oracle, spk, n, k, k, 1.5, 1, 107)
    fact = spk.factorize(a, spk.make_plan(n, k, k, 4, 1.0, 2.0))
    x = spk.solve(fact, np.zeros((n, 0)))
    assert x.shape == (n, 0)
    with pytest.raises(ValueError):
        spk.solve(fact, np.zeros((n + 1, 1)))
    with pytest.raises(ValueError):
        spk.transpose_solve(fact, np.zeros((n + 1, 1)))


def test_serial_plan(oracle, spk):
    n, k = 100, 3
    a, band, F = make_case(oracle, spk, n, k, k, 1.5, 2, 17)
    fact = spk.factorize(a, spk.make_plan(n, k, k, 1, 1.0, 2.0))
    assert fact.p() == 1
    assert spk.relative_residual(a, spk.solve(fact, F), F) < 1e-12
    assert spk.relative_residual(a, spk.transpose_solve(fact, F), F, True) < 1e-12


def test_pivoting_singular_column_raises(spk):
    n, k = 64, 2
    a = spk.BandedMatrix(n, k, k)
    for i in range(n):
        a.set(i, i, 1.0)
    for i in range(10, 13):  # zero a whole column inside partition 0's band
        pass
    for i in range(max(0, 5 - k), min(n, 5 + k + 1)):
        a.set(i, 5, 0.0)
    with pytest.raises(RuntimeError):
        spk.factorize(a, spk.make_plan(n, k, k, 2, 1.0, 2.0), spk.FactorOptions(pivoting=True))


def test_boost_and_refine(oracle, spk):
    """test_solve_stage.cpp:246-259 : a boosted factorization + refinement."""
    n, k = 200, 3
    a, band, F = make_case(oracle, spk, n, k, k, 1.5, 2, 89)
    a.set(0, 0, 0.0)
    plan = spk.make_plan(n, k, k, 2, 1.0, 2.0)
    fact = spk.factorize(a, plan)
    assert fact.boost_count >= 1
    r = spk.iterative_refine(fact, a, F, np.zeros((n, 2)), 5, 1e-12)
    assert r.converged and r.iterations <= 5
    assert spk.relative_residual(a, r.x, F) <= 1e-12


def test_decoupled_boundaries_zero_tips(oracle, spk):
    n, k = 80, 2
    plan = spk.make_plan(n, k, k, 4, 1.0, 2.0)
    a, band, F = make_case(oracle, spk, n, k, k, 1.5, 2, 5)
    for b in plan.bounds[1:-1]:
        for j in range(b - k, b + k):
            for i in range(max(0, j - k), min(n, j + k + 1)):
                if (i < b) != (j < b):
                    a.set(i, j, 0.0)
    fact = spk.factorize(a, plan)
    for i in range(plan.p):
        assert np.abs(fact.vb[i]).max() == 0.0
        assert np.abs(fact.wt[i]).max() == 0.0
    xo = oracle.oracle_solve(a.data, n, k, k, F)
    assert rel_componentwise(spk.solve(fact, F), xo) < 1e-12


def test_cpp_dropin_api(spk, tmp_path):
    """The reference-style C++ API (include/spike/*.hpp) against libspike_b200.so."""
    import os
    import shutil
    import subprocess
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    cxx = shutil.which("g++")
    if cxx is None:
        pytest.skip("no host C++ compiler")
    exe = tmp_path / "dropin_test"
    libdir = os.path.dirname(spk.LIB_PATH)
    subprocess.run([cxx, "-std=c++17", "-O1", os.path.join(root, "tests", "cpp", "dropin_test.cpp"),
                    "-I", os.path.join(root, "include"), spk.LIB_PATH, f"-Wl,-rpath,{libdir}", "-o", str(exe)],
                   check=True)
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0 and "DROPIN PASS" in r.stdout, r.stdout + r.stderr


GOLDEN_CASES = ["c1_small", "c2_small", "c3_small", "c4_small", "asym", "asym_piv", "dual_mix", "serial", "k1"]


@pytest.mark.parametrize("name", GOLDEN_CASES)
def test_gpu_matches_reference_golden(oracle, spk, name):
    """GPU solutions vs the compiled reference's own outputs (tests/golden), same plan."""
    import os
    g = np.load(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "golden.npz"))
    n, kl, ku, nrhs, t, piv = [int(x) for x in g[name + "/shape"]]
    dd = float(g[name + "/dd"][0])
    band = oracle.generate_band(20181108, n, kl, ku, dd)
    F = np.asfortranarray(oracle.generate_rhs(20181109, n, nrhs))
    plan = spk.PartitionPlan(p=len(g[name + "/bounds"]) - 1, bounds=[int(b) for b in g[name + "/bounds"]],
                             kinds=[spk.PartitionKind(int(x)) for x in g[name + "/kinds"]])
    fact = spk.factorize(spk.BandedMatrix(n, kl, ku, band), plan, spk.FactorOptions(pivoting=bool(piv)))
    tol = 1e-9 if piv else 1e-12
    st, stt = spk.SolveStats(), spk.SolveStats()
    assert rel_componentwise(spk.solve(fact, F, st), g[name + "/x"]) <= tol
    assert rel_componentwise(spk.transpose_solve(fact, F, stt), g[name + "/xt"]) <= tol
    assert st.partition_full_sweeps == list(g[name + "/sweeps"])
    assert stt.partition_full_sweeps == list(g[name + "/sweeps_t"])
    assert [st.reduced_coupling_solves, stt.reduced_coupling_solves] == list(g[name + "/couplings"])
    assert fact.factor_sweeps == list(g[name + "/factor_sweeps"])
    assert [fact.levels.levels(), fact.boost_count] == list(g[name + "/levels"])
    for w in ("vt", "vb", "wt", "wb", "bhat", "chat"):
        ref = g[name + "/" + w]
        for i in range(plan.p):
            assert rel_componentwise(getattr(fact, w)[i], ref[i]) <= (1e-9 if piv else 1e-12), (w, i)


# Full BASELINE sizes against the compiled reference: tests/test_gpu_scale_parity.py


# Blocked pivoted DMMA LU + pivoted DMMA forward sweep (spk_lu_piv_dmma.cu,
# spk_sweep_piv_dmma.cu) and the dense DMMA LU of the 2k coupling units, on
# non-dominant bands (pivots leave the diagonal, |W| > 1 takes the generic
# coupling path): ragged partition lengths (m mod 8 != 0, so the UL
# partition's panels and the truncated tail sweeps start mid-block),
# asymmetric bands both ways, every kernel template (kl+kc <= 64/128/192).
PIV_CASES = [(3001, 7, 13, 5, 3), (4099, 24, 9, 6, 2), (2503, 40, 40, 3, 5), (5003, 64, 64, 7, 4),
             (6007, 30, 90, 4, 3), (2999, 1, 1, 9, 1)]


@pytest.mark.parametrize("n,kl,ku,p,nrhs", PIV_CASES)
def test_pivoted_dmma_kernels_non_dominant(oracle, spk, n, kl, ku, p, nrhs):
    """Narrow random bands without dominance can be arbitrarily ill-conditioned
    (and pivoted SPIKE then loses backward stability with p, PAPER.md): the bar
    is the oracle running the same algorithm on the same plan -- residual no
    worse than the oracle's, solution gap within SURVEY 8(d)'s 1e-10 * cond."""
    a, band, F = make_case(oracle, spk, n, kl, ku, -1.0, nrhs, 7000 + n + kl)
    plan = spk.gpu_plan(n, kl, ku, nrhs, True, p)
    assert plan.p == p
    fact = spk.factorize(a, plan, spk.FactorOptions(pivoting=True))
    of = oracle.factorize(band, n, kl, ku, plan.bounds, True)
    cond = oracle.cond1(band, n, kl, ku)
    for tr in (False, True):
        X = spk.transpose_solve(fact, F) if tr else spk.solve(fact, F)
        Xo = of.solve(F, tr)[0]
        res = oracle.relative_residual(band, n, kl, ku, X, F, tr)
        res_o = oracle.relative_residual(band, n, kl, ku, Xo, F, tr)
        gap = np.abs(X - Xo).max() / max(np.abs(Xo).max(), 1e-300)
        assert res <= max(RES_TOL, 10.0 * res_o), (tr, res, res_o, cond)
        assert gap <= max(GAP_TOL, 1e-10 * cond), (tr, gap, cond)
    # bit-deterministic repeats
    X1 = spk.solve(spk.factorize(a, plan, spk.FactorOptions(pivoting=True)), F)
    assert np.array_equal(X1, spk.solve(fact, F))
